"""Summarize gpurun_out/<tag>_* ncu outputs into profiles/ (tracked)."""
import csv, collections, io, json, os, subprocess, sys

tag = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 512
dim = int(sys.argv[3]) if len(sys.argv) > 3 else 3
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
go = os.path.join(root, "gpurun_out")
prof = os.environ.get("PROF_OUT", os.path.join(root, "profiles"))
os.makedirs(prof, exist_ok=True)
out = []

# ---- launch list
rows = list(csv.reader(open(os.path.join(go, f"{tag}_launches.csv"))))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
L = {}
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    d = L.setdefault(int(r[idi]), {"name": r[ki]})
    d[r[mi]] = float(r[vi].replace(",", ""))
tot = collections.defaultdict(lambda: [0, 0.0, 0.0])
fine_sweeps = []
for k in sorted(L):
    d = L[k]
    nm = d["name"].split("(")[0].replace("void ", "").replace("fasmg::", "")
    if nm.startswith("at::"):
        continue  # torch input generation in the profiling script, not the solver
    key = nm.split("<")[0]
    t = d.get("gpu__time_duration.sum", 0.0)
    by = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    tot[key][0] += 1
    tot[key][1] += t
    tot[key][2] += by
    # plain half-sweeps only: the corrected one (template flag true / 1) is a
    # different kernel with its own coarse reads
    full = d["name"]
    corr = ", 1>(" in full or ", true>(" in full or "(bool)1>" in full
    if key.startswith("k_sweep_tma") and t > 0 and not corr:
        fine_sweeps.append((t, by))
alltime = sum(v[1] for v in tot.values())
out.append(f"# {tag}: ncu launch list of one eager V-cycle + norm, 3D {n}^3 heat "
           f"(gpu__time_duration, cold-cache serialized; compare SHARES)")
out.append(f"{'kernel':24s} {'launches':>8s} {'time_ms':>9s} {'share':>6s} {'dram_GB':>8s} {'GB/s':>7s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1][1]):
    out.append(f"{k:24s} {v[0]:8d} {v[1]/1e6:9.3f} {100*v[1]/alltime:5.1f}% {v[2]/1e9:8.3f} "
               f"{(v[2]/v[1] if v[1] else 0):7.0f}")
out.append(f"total fasmg kernel time {alltime/1e6:.3f} ms")
# finest-level sweeps = the largest ones
fine_sweeps.sort(key=lambda x: -x[0])
top = [x for x in fine_sweeps if x[0] >= 0.5 * fine_sweeps[0][0]]
avg_t = sum(x[0] for x in top) / len(top)
avg_b = sum(x[1] for x in top) / len(top)
alg = 12.0 * n ** dim
out.append(f"finest plain half-sweeps: {len(top)} launches, mean {avg_t/1e3:.1f} us, dram {avg_b/1e9:.3f} GB "
           f"per launch (algorithmic {alg/1e9:.3f} GB, ratio {avg_b/alg:.3f}), "
           f"share of fasmg time {100*sum(x[0] for x in top)/alltime:.1f}%")
json.dump({"tag": tag, "n": n, "dim": dim, "dram_bytes_per_launch": avg_b,
           "algorithmic_bytes_per_launch": alg, "ncu_time_us": avg_t / 1e3,
           "source": f"gpurun_out/{tag}_launches.csv (ncu --metrics dram__bytes_read.sum,"
                     "dram__bytes_write.sum)"},
          open(os.path.join(prof, "ncu_sweep_traffic.json"), "w"), indent=1)

# ---- full captures
def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    return dict(zip(r[0], r[2])), dict(zip(r[0], r[1]))

want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
for kind in ("sweep", "tau", "corr", "etau", "spec", "ecorr"):
    rep = os.path.join(go, f"{tag}_{kind}.ncu-rep")
    if not os.path.exists(rep):
        continue
    v, u = raw(rep)
    label = {"sweep": "finest half-sweep (k_sweep_tma)", "tau": "finest tau pass (k_resid_tma<1>)",
             "corr": "finest corrected half-sweep (k_sweep_tma<.., CORR>)",
             "etau": "finest edge-field tau pass (k_tau_edge_tma, EDGE_NS)",
             "spec": "outer norm + next first half-sweep (k_resid_tma<2>)",
             "ecorr": "finest edge corrected half-sweep (k_sweep_tma<EA, M, CORR>, EDGE_NS)"}[kind]
    out.append(f"\n# {tag}: ncu --set full, one launch: {label}")
    for k in want:
        if k in v:
            out.append(f"{k:60s} {v[k]} {u.get(k, '')}")
    stalls = {k: v[k] for k in v if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    top = sorted(((float(x.replace(",", "")), k) for k, x in stalls.items() if x), reverse=True)[:5]
    out.append("top stall samples: " + ", ".join(f"{k.split('stalled_')[1]}={int(c)}" for c, k in top))
txt = "\n".join(out) + "\n"
open(os.path.join(prof, f"{tag}_ncu_summary.txt"), "w").write(txt)
print(txt)
