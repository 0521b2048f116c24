cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ad; mkdir -p $O
timeout 1500 python -m pytest tests/test_wave_gpu.py tests/test_gpu_parity.py tests/test_ns_gpu.py tests/test_fullsize_gpu.py -q -x 2>&1 | tail -2 > $O/tests.log
for l in ns ew tb; do timeout 300 python scripts/vcycle_prof.py 512 $l 5 > $O/prof_${l}.txt 2>&1; done
FASMG_CORR_WALK=0 timeout 300 python scripts/vcycle_prof.py 512 ns 5 > $O/prof_ns_nowalk.txt 2>&1
timeout 900 python bench.py --workload ns512 --steps 5 --warmup 3 --no-cpu-baseline > $O/ns512.json 2> $O/ns512.err
