python __graft_entry__.py build
python scripts/initcheck_probe.py ns; echo "plain ns rc=$?"
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 600 $CS --tool memcheck python scripts/initcheck_probe.py ns 2>&1 | tail -30; echo "memcheck ns"
