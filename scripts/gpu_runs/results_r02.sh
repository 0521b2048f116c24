# refresh results/ (round 2 code): CLI timing tables, NS 512^3 schemes, V-cycle by size/location
cd $GRAFT_REPO_ROOT
O=gpurun_out/results_r02; mkdir -p $O
timeout 900 python -m paper_2510_11152_b200 timing --dim 3 --size 64,128,256,512 --out $O/timing_3d.csv > $O/timing_3d.log 2>&1
timeout 900 python -m paper_2510_11152_b200 timing --dim 2 --size 1024,2048,4096,8192,16384 --out $O/timing_2d.csv > $O/timing_2d.log 2>&1
timeout 900 python scripts/probe_perf.py 512x3 1024x3 8192x2 16384x2 > $O/vcycle_sizes.txt 2>&1
for l in cell ew ns tb; do timeout 300 python scripts/vcycle_prof.py 512 $l 5 2>&1 | grep live >> $O/vcycle_by_location_512.txt; done
timeout 900 python scripts/ns_perf.py 512 2 4 efficient > $O/ns512_order2_efficient.json 2> $O/ns.err
timeout 900 python scripts/ns_perf.py 512 2 4 classical > $O/ns512_order2_classical.json 2>> $O/ns.err
timeout 900 python scripts/ns_perf.py 512 1 4 efficient > $O/ns512_order1_efficient.json 2>> $O/ns.err
