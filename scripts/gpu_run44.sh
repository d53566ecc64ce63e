# L2 residency experiment: evict-first threshold 32 MB (default) vs 256 MB on the 1M-DOF 2D configs.
python __graft_entry__.py build
for mb in 32 256; do
for cfg in td_l10 c2; do
MGB200_STREAM_MB=$mb timeout 900 python bench.py --config $cfg --steps 10 --no-cpu-baseline --no-mixed > gpurun_out/b44.json 2> gpurun_out/b44.err
python -c "import json; d=json.load(open('gpurun_out/b44.json')); print('$mb', '$cfg', round(d['value'],1), round(d['solve_ms'],3), round(d['vcycle_only']['ms'],4), round(d['roofline']['avg_launch_ms']*1e3,1), round(d['spmv_hbm']['avg_launch_ms']*1e3,1))"
done; done
