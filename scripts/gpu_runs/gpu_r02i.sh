cd $GRAFT_REPO_ROOT
O=gpurun_out/r02i; mkdir -p $O
timeout 600 python -m pytest tests/test_wave_gpu.py -q -x 2>&1 | tail -30 > $O/wave_tests.log
timeout 300 python scripts/level_sweep_scan.py "" "FASMG_PAIR=0" "FASMG_PAIR_CHUNK=4" "FASMG_PAIR_CHUNK=16" > $O/scan.txt 2>&1
timeout 300 python scripts/vcycle_prof.py 512 cell 5 $O/prof_cell.json > $O/prof_cell.txt 2>&1
