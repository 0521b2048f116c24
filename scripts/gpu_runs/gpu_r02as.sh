cd $GRAFT_REPO_ROOT
O=gpurun_out/r02as; mkdir -p $O
ncu --set full --clock-control none --import-source on -k regex:k_sweep_tma -s 24 -c 1 \
    -o $O/ecorr python scripts/profile_vcycle.py 512 3 1 edge_ns > $O/ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sweep_tma -s 2 -c 1 \
    -o $O/esweep python scripts/profile_vcycle.py 512 3 1 edge_ns > $O/ncu2.log 2>&1
for k in ecorr esweep; do
ncu -i $O/$k.ncu-rep --page details --csv > $O/${k}_details.csv 2>/dev/null
ncu -i $O/$k.ncu-rep --page source --csv --print-source cuda,sass > $O/${k}_source.csv 2>/dev/null
done
gzip -f $O/*_source.csv; rm -f $O/*.ncu-rep
