cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ao; mkdir -p $O
timeout 900 python -m pytest tests/test_wave_gpu.py -q -x -k "edge_fused" 2>&1 | tail -30 > $O/tests.log
timeout 1200 python -m pytest tests/test_wave_gpu.py tests/test_gpu_parity.py tests/test_ns_gpu.py -q 2>&1 | tail -30 > $O/tests2.log
for l in ew tb ns; do timeout 300 python scripts/vcycle_prof.py 512 $l 5 > $O/prof_${l}.txt 2>&1; done
