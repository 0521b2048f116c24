cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ah; mkdir -p $O
timeout 1500 python -m pytest tests/test_slab_gpu.py tests/test_ns_slab_gpu.py -q -x 2>&1 | tail -2 > $O/tests.log
timeout 600 python scripts/virtual_slab_perf.py 512 1 2 4 8 > $O/vperf.txt 2>&1
FASMG_RESID_TMA=0 timeout 600 python scripts/virtual_slab_perf.py 512 2 4 8 > $O/vperf_noresid.txt 2>&1
