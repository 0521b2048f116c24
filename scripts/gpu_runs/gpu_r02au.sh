cd $GRAFT_REPO_ROOT
O=gpurun_out/r02au; mkdir -p $O
timeout 900 python -m pytest tests/test_wave_gpu.py -q -x -k "edge_fused" 2>&1 | tail -3 > $O/tests.log
for c in 4 8 16; do FASMG_CORR_CHUNK=$c timeout 300 python scripts/vcycle_prof.py 512 ew 5 > $O/prof_ew_c$c.txt 2>&1; done
