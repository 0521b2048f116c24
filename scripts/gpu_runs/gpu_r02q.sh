cd $GRAFT_REPO_ROOT
O=gpurun_out/r02q; mkdir -p $O
timeout 900 python -m pytest tests/test_wave_gpu.py -q -k edge_tau 2>&1 | tail -3 > $O/tests.log
for ch in 4 8 16; do for l in ns ew; do FASMG_ETAU_CHUNK=$ch timeout 300 python scripts/vcycle_prof.py 512 $l 5 > $O/prof_${l}_$ch.txt 2>&1; done; done
