cd $GRAFT_REPO_ROOT
O=gpurun_out/r02l; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider 2>&1 | tail -8 > $O/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 300 python scripts/vcycle_prof.py 512 cell 5 $O/prof_cell.json > $O/prof_cell.txt 2>&1
timeout 300 python scripts/vcycle_prof.py 512 ns 5 $O/prof_ns.json > $O/prof_ns.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sweep_tma -s 24 -c 1 -o $O/corr python scripts/profile_vcycle.py 512 3 1 > $O/ncu.log 2>&1
