cd $GRAFT_REPO_ROOT
O=gpurun_out/r02az; mkdir -p $O
timeout 600 python scripts/ns_prof.py 512 2 2 > $O/nsprof.txt 2>&1
timeout 300 python scripts/vcycle_prof.py 512 cell 5 > $O/prof_cell.txt 2>&1
FASMG_NORM_SMEM=80000 timeout 300 python scripts/vcycle_prof.py 512 cell 5 > $O/prof_cell_n80.txt 2>&1
