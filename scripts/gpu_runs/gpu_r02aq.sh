cd $GRAFT_REPO_ROOT
O=gpurun_out/r02aq; mkdir -p $O
ncu --set full --clock-control none --import-source on -k regex:k_sweep_tma -s 24 -c 1 \
    -o $O/ecorr python scripts/profile_vcycle.py 512 3 1 edge_ns > $O/ncu.log 2>&1
ncu -i $O/ecorr.ncu-rep --page details --csv > $O/ecorr_details.csv 2>/dev/null
ncu -i $O/ecorr.ncu-rep --page source --csv --print-source cuda,sass > $O/ecorr_source.csv 2>/dev/null
gzip -f $O/ecorr_source.csv; rm -f $O/*.ncu-rep
