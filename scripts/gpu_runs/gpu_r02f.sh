cd $GRAFT_REPO_ROOT
O=gpurun_out/r02f; mkdir -p $O
timeout 200 python scripts/ns_slab_debug.py 64 4 2 > $O/ns64_4.log 2>&1; echo "rc=$?" >> $O/ns64_4.log
timeout 1200 python -m pytest tests/test_ns_slab_gpu.py tests/test_slab_gpu.py -q 2>&1 | tail -15 > $O/tests.log
