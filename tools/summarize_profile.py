"""Summarise gpurun_out/{launches.csv, prof_iter.ncu-rep, bench*.json} into profiles/<tag>_*.

usage: python tools/summarize_profile.py r1_config3
"""
import collections, csv, json, os, subprocess, sys

tag = sys.argv[1]
cfg_id = sys.argv[2] if len(sys.argv) > 2 else "5"
G = "gpurun_out"
os.makedirs("profiles", exist_ok=True)
out = [f"# ncu summary {tag}\n"]

# launch list (metrics pass: gpu__time_duration, cold cache, serialised)
rows = list(csv.reader(open(os.path.join(G, "launches.csv"))))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
iname, ival, iunit = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) > ival:
        agg[r[iname]].append(float(r[ival].replace(",", "")))
unit = rows[hi + 1][iunit]
out.append("## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`)\n")
out.append("Cold-cache, serialised per-launch times: compare shares, not absolutes.\n")
out.append("| kernel | launches | mean | share of one iteration (K4+K4b+K2+K3) |")
out.append("|---|---|---|---|")
it_kernels = {k: sum(v) / len(v) for k, v in agg.items() if any(x in k for x in ("k_yg", "k_zx", "k_r_tma<1>", "k_r<1", "k_sel_greedy"))}
it_total = sum(it_kernels.values())
for k, v in agg.items():
    mean = sum(v) / len(v)
    share = f"{mean / it_total:.3f}" if k in it_kernels else ""
    out.append(f"| `{k[:60]}` | {len(v)} | {mean / 1000:.2f} us | {share} |")
with open(os.path.join("profiles", f"{tag}_launches.csv"), "w") as f:
    f.writelines(",".join(r) + "\n" for r in rows[hi:])

# full capture
raw = subprocess.run(["ncu", "-i", os.path.join(G, "prof_iter.ncu-rep"), "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout.splitlines()
rr = list(csv.reader(raw))
hh, units = rr[0], rr[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_active.avg", "sm__cycles_elapsed.avg", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic",
        "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum",
        "lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum"]
out.append("\n## `ncu --set full` (one launch each)\n")
out.append("| metric | " + " | ".join(r[hh.index("Kernel Name")][:40] for r in rr[2:]) + " |")
out.append("|---|" + "---|" * (len(rr) - 2))
summary = {}
for w in want:
    if w in hh:
        i = hh.index(w)
        out.append(f"| {w} ({units[i]}) | " + " | ".join(r[i] for r in rr[2:]) + " |")
for r in rr[2:]:
    name = r[hh.index("Kernel Name")]
    summary[name] = {w: r[hh.index(w)] for w in want if w in hh}
    summary[name]["_units"] = {w: units[hh.index(w)] for w in want if w in hh}
json.dump(summary, open(os.path.join("profiles", f"{tag}_ncu_full.json"), "w"), indent=1)
# K2 traffic per launch (bytes) for bench.py's roofline.traffic
for name, d in summary.items():
    if "k_r_tma<1>" in name or "k_r_tma<(bool)1>" in name:
        mult = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0}
        rd = float(d["dram__bytes_read.sum"]) * mult[d["_units"]["dram__bytes_read.sum"]]
        wr = float(d["dram__bytes_write.sum"]) * mult[d["_units"]["dram__bytes_write.sum"]]
        json.dump({"dram_bytes_per_launch": rd + wr, "read": rd, "write": wr,
                   "source": f"profiles/{tag}_ncu_full.json (ncu --set full, one launch)"},
                  open(os.path.join("profiles", f"k2_traffic_config{cfg_id}.json"), "w"), indent=1)
for b in ("bench.json", "bench_ref.json"):
    p = os.path.join(G, b)
    if os.path.exists(p):
        txt = open(p).read().strip()
        open(os.path.join("profiles", f"{tag}_{b}"), "w").write(txt + "\n")
        out.append(f"\n## {b}\n\n```json\n{txt}\n```")
open(os.path.join("profiles", f"{tag}_summary.md"), "w").write("\n".join(out) + "\n")
print("\n".join(out[:40]))
