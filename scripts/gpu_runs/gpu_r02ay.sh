cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ay; mkdir -p $O
timeout 300 python scripts/vcycle_prof.py 512 cell 5 > $O/prof_base.txt 2>&1
cp gpurun_varA.so paper_2510_11152_b200/libfasmg_b200.so
timeout 300 python scripts/vcycle_prof.py 512 cell 5 > $O/prof_A58.txt 2>&1
FASMG_NORM_SMEM=49200 timeout 300 python scripts/vcycle_prof.py 512 cell 5 > $O/prof_A49.txt 2>&1
timeout 600 python -m pytest tests/test_wave_gpu.py -q -x -k "speculative" 2>&1 | tail -2 > $O/testsA.log
