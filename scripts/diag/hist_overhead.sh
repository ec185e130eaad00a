cd $GRAFT_REPO_ROOT
for n in 1212416 4000000000; do timeout 300 python scripts/c4_perf.py --hist-n $n --km-n 0 --steps 5 2>&1 | grep histogram; done
