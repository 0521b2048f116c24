cd $GRAFT_REPO_ROOT
O=gpurun_out/r02am; mkdir -p $O
timeout 900 python -m pytest tests/test_wave_gpu.py -q -x -k "speculat" 2>&1 | tail -15 > $O/spec_tests.log
timeout 1500 python -m pytest tests/test_wave_gpu.py tests/test_gpu_parity.py tests/test_fullsize_gpu.py tests/test_heat_gpu.py tests/test_batch_gpu.py tests/test_arena_gpu.py -q -x 2>&1 | tail -3 > $O/tests.log
timeout 300 python scripts/vcycle_prof.py 512 cell 5 > $O/prof_cell.txt 2>&1
FASMG_SPEC=0 timeout 300 python scripts/vcycle_prof.py 512 cell 5 > $O/prof_cell_nospec.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-numba-baseline > $O/bench.json 2> $O/bench.err
