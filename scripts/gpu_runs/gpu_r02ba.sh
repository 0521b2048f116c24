cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ba; mkdir -p $O
for c in 4 2 3; do FASMG_CHUNK_L1=$c timeout 300 python scripts/vcycle_prof.py 512 cell 5 > $O/prof_cell_$c.txt 2>&1; done
for c in 4 2; do FASMG_CHUNK_L1=$c timeout 300 python scripts/vcycle_prof.py 512 ew 5 > $O/prof_ew_$c.txt 2>&1; done
