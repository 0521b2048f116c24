cd $GRAFT_REPO_ROOT
O=gpurun_out/r02aw; mkdir -p $O
# variant B (built in place: CORR bound 3) then variant A (cell CORR bound 4)
timeout 600 python -m pytest tests/test_wave_gpu.py -q -x -k "fused_correction" 2>&1 | tail -2 > $O/testsB.log
for c in 4 8 16; do FASMG_CORR_CHUNK=$c timeout 300 python scripts/vcycle_prof.py 512 cell 5 > $O/profB_c$c.txt 2>&1; done
cp gpurun_varA.so paper_2510_11152_b200/libfasmg_b200.so
timeout 600 python -m pytest tests/test_wave_gpu.py -q -x -k "fused_correction" 2>&1 | tail -2 > $O/testsA.log
for c in 4 8 16; do FASMG_CORR_CHUNK=$c timeout 300 python scripts/vcycle_prof.py 512 cell 5 > $O/profA_c$c.txt 2>&1; done
