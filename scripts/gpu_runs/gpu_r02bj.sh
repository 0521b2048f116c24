cd $GRAFT_REPO_ROOT
O=gpurun_out/r02bj; mkdir -p $O
timeout 1800 python -m pytest tests -q -m gpu -x 2>&1 | tail -3 > $O/tests.log
for l in ew cell; do timeout 300 python scripts/vcycle_prof.py 512 $l 5 > $O/prof_$l.txt 2>&1; done
