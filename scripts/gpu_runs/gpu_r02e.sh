cd $GRAFT_REPO_ROOT
O=gpurun_out/r02e; mkdir -p $O
run() { name=$1; shift; timeout 100 "$@" > $O/$name.log 2>&1; echo "rc=$?" >> $O/$name.log; }
run v64_4_neu python scripts/virtual_slab_case.py 64 4 neumann cell
run v64_4_dir python scripts/virtual_slab_case.py 64 4 dirichlet cell
run v64_2_neu python scripts/virtual_slab_case.py 64 2 neumann cell
run v128_4_neu python scripts/virtual_slab_case.py 128 4 neumann cell
run v64_4_ew python scripts/virtual_slab_case.py 64 4 dirichlet edge_ew
run ns64_4_c32 env CUDA_DEVICE_MAX_CONNECTIONS=32 python scripts/ns_slab_debug.py 64 4 2
run ns64_2 python scripts/ns_slab_debug.py 64 2 2
SELFTEST_N=64 SELFTEST_BC=neumann timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29656 scripts/dist_selftest.py > $O/dist4_neu.log 2>&1; echo "rc=$?" >> $O/dist4_neu.log
timeout 600 python -m pytest tests/test_wave_gpu.py -q -x 2>&1 | tail -5 > $O/wave_tests.log
