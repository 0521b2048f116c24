cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ax; mkdir -p $O
# variant B (in place: edge CORR with TMA f boxes), then A (f from global)
timeout 600 python -m pytest tests/test_wave_gpu.py -q -x -k "fused_correction" 2>&1 | tail -2 > $O/testsB.log
for l in ew cell; do timeout 300 python scripts/vcycle_prof.py 512 $l 5 > $O/profB_$l.txt 2>&1; done
cp gpurun_varA.so paper_2510_11152_b200/libfasmg_b200.so
for l in ew cell; do timeout 300 python scripts/vcycle_prof.py 512 $l 5 > $O/profA_$l.txt 2>&1; done
