cd $GRAFT_REPO_ROOT
O=gpurun_out/r02bm; mkdir -p $O
timeout 300 python scripts/vcycle_prof.py 512 cell 5 > $O/prof_base.txt 2>&1
for v in "FASMG_NORM_CHUNK=2" "FASMG_NORM_CHUNK=8" "FASMG_TAU_CHUNK=2" "FASMG_TAU_CHUNK=8" "FASMG_CORR_CHUNK=16" "FASMG_CORR_CHUNK=6"; do
  env $v timeout 300 python scripts/vcycle_prof.py 512 cell 5 > $O/prof_$v.txt 2>&1
done
