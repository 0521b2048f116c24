cd $GRAFT_REPO_ROOT
O=gpurun_out/r02d; mkdir -p $O
timeout 120 python scripts/ns_slab_debug.py 32 4 2 > $O/dbg_32_4.log 2>&1; echo rc=$? >> $O/dbg_32_4.log
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 120 python scripts/ns_slab_debug.py 32 4 2 > $O/dbg_32_4_c32.log 2>&1; echo rc=$? >> $O/dbg_32_4_c32.log
timeout 120 python scripts/ns_slab_debug.py 64 4 2 > $O/dbg_64_4.log 2>&1; echo rc=$? >> $O/dbg_64_4.log
timeout 900 python -m pytest tests/test_ns_slab_gpu.py -q -k "not fill" 2>&1 | tail -15 > $O/tests.log
