cd $GRAFT_REPO_ROOT
O=gpurun_out/r02j; mkdir -p $O
timeout 600 python -m pytest tests/test_wave_gpu.py -q 2>&1 | tail -12 > $O/wave_tests.log
timeout 300 python scripts/level_sweep_scan.py "" "FASMG_PAIR=0" "FASMG_PAIR_CHUNK=4" "FASMG_PAIR_CHUNK=16" > $O/scan.txt 2>&1
timeout 300 python scripts/vcycle_prof.py 512 cell 5 $O/prof_cell.json > $O/prof_cell.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pair_tma -s 2 -c 1 -o $O/pair python scripts/profile_vcycle.py 512 3 1 > $O/ncu.log 2>&1
