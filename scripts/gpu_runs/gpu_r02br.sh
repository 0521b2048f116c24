cd $GRAFT_REPO_ROOT
O=gpurun_out/r02br; mkdir -p $O
timeout 1800 python -m pytest tests -q -m gpu -x -p no:cacheprovider 2>&1 | tail -3 > $O/tests.log
for l in ew cell; do timeout 300 python scripts/vcycle_prof.py 512 $l 5 > $O/prof_$l.txt 2>&1; done
timeout 900 python bench.py --workload ns512 --steps 5 --warmup 3 --no-cpu-baseline > $O/ns512.json 2> $O/ns512.err
