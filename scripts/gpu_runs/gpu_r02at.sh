cd $GRAFT_REPO_ROOT
O=gpurun_out/r02at; mkdir -p $O
timeout 900 python -m pytest tests/test_wave_gpu.py -q -x -k "edge_fused or fused_correction" 2>&1 | tail -30 > $O/tests.log
for l in ew ns tb; do timeout 300 python scripts/vcycle_prof.py 512 $l 5 > $O/prof_${l}.txt 2>&1; done
FASMG_CORR_CHUNK=16 timeout 300 python scripts/vcycle_prof.py 512 ew 5 > $O/prof_ew_c16.txt 2>&1
FASMG_CORR_CHUNK=4 timeout 300 python scripts/vcycle_prof.py 512 ew 5 > $O/prof_ew_c4.txt 2>&1
