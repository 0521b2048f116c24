cd $GRAFT_REPO_ROOT
O=gpurun_out/r02aa; mkdir -p $O
timeout 900 python -m pytest tests/test_wave_gpu.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2 > $O/tests.log
timeout 600 python scripts/level_sweep_scan.py "FASMG_RESID_PF=0" "" "FASMG_RESID_PF=0" "" > $O/scan.txt 2>&1
timeout 300 python scripts/vcycle_prof.py 512 cell 5 > $O/prof_cell.txt 2>&1
FASMG_RESID_PF=0 timeout 300 python scripts/vcycle_prof.py 512 cell 5 > $O/prof_cell_nopf.txt 2>&1
timeout 300 python scripts/vcycle_prof.py 512 ns 5 > $O/prof_ns.txt 2>&1
