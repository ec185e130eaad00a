python scripts/c4_perf.py --hist-n 1048576 --km-n 200000000 --steps 2 2>&1 | grep kmeans_assign | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['kernel_ms'],2))"
