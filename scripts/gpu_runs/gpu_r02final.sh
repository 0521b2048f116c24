#!/bin/bash
# final state: GPU suite, smoke, bench (1 GPU), reference arm, NS 512^3
cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-r02f}; mkdir -p $O
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/gpu_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference > $O/ref.json 2>> $O/bench.err
timeout 900 python bench.py --workload ns512 --steps 5 --warmup 3 > $O/ns512.json 2>> $O/bench.err
