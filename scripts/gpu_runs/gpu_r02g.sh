cd $GRAFT_REPO_ROOT
O=gpurun_out/r02g; mkdir -p $O
timeout 600 python -m pytest tests/test_slab_gpu.py -q -k four 2>&1 | tail -3 > $O/four.log
for loc in cell ns; do timeout 300 python scripts/vcycle_prof.py 512 $loc 5 $O/prof_$loc.json > $O/prof_$loc.txt 2>&1; done
