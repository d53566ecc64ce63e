#!/bin/bash
# round 2 profiles: launch list of one C3 bench step (DRAM bytes per launch), --set full of the
# fine-level kernels, the bench.py launch list itself, and bench lines (C3 full, C5, C2).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2i_build.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2i_c3_step.csv python scripts/profile_ops.py step --config c3 > gpurun_out/r2i_step.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -o gpurun_out/r2i_c3_full python scripts/profile_ops.py kernels --config c3 > gpurun_out/r2i_full.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 3200 -c 1200 --csv --log-file gpurun_out/r2i_bench_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-mixed > gpurun_out/r2i_bench_under_ncu.log 2>&1
timeout 1500 python bench.py > gpurun_out/r2i_c3.json 2> gpurun_out/r2i_c3.err
timeout 900 python bench.py --config c5 --no-cpu-solve > gpurun_out/r2i_c5.json 2> gpurun_out/r2i_c5.err
timeout 900 python bench.py --config c2 > gpurun_out/r2i_c2.json 2> gpurun_out/r2i_c2.err
timeout 900 python bench.py --impl reference > gpurun_out/r2i_ref.json 2> gpurun_out/r2i_ref.err
