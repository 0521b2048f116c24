cd $GRAFT_REPO_ROOT
O=gpurun_out/r02bd; mkdir -p $O
for m in 2097152 262144 32768; do FASMG_TMA_MIN=$m timeout 300 python scripts/vcycle_prof.py 512 cell 5 > $O/prof_cell_$m.txt 2>&1; done
for m in 2097152 262144; do FASMG_TMA_MIN=$m timeout 300 python scripts/vcycle_prof.py 512 ew 5 > $O/prof_ew_$m.txt 2>&1; done
