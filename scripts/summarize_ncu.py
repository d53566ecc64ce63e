"""Summarise ncu outputs from gpurun_out/ into committed profiles/ files.

usage: python scripts/summarize_ncu.py <tag> <launches.csv> [<full.ncu-rep>] [--config c3]
writes profiles/<tag>_launches.csv (per launch: id, kernel, grid, ns, dram bytes),
       profiles/<tag>_summary.md (per-kernel shares of one step + full-capture metrics),
       profiles/ncu_traffic.json (fine-level sweep DRAM bytes per launch, read by bench.py).
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
FULL_METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
                "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
                "smsp__inst_executed.sum", "launch__grid_size", "sm__cycles_elapsed.avg.per_second",
                "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]


def short(name):
    return name.split("(")[0].replace("void ", "").replace("mgk::", "")


def read_launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    gi = h.index("Grid Size")
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        d = per.setdefault(int(r[ii]), {"kernel": r[ki], "grid": r[gi]})
        d[r[mi]] = float(r[vi].replace(",", ""))
    return per


def main():
    tag, lcsv = sys.argv[1], sys.argv[2]
    rep = sys.argv[3] if len(sys.argv) > 3 and sys.argv[3].endswith(".ncu-rep") else None
    config = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else "c3"
    os.makedirs(PROF, exist_ok=True)
    per = read_launches(lcsv)
    with open(os.path.join(PROF, f"{tag}_launches.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["id", "kernel", "grid", "gpu_time_ns", "dram_read_bytes", "dram_write_bytes"])
        for i, d in per.items():
            w.writerow([i, short(d["kernel"]), d["grid"], int(d.get("gpu__time_duration.sum", 0)),
                        int(d.get("dram__bytes_read.sum", 0)), int(d.get("dram__bytes_write.sum", 0))])
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    tot = 0.0
    for d in per.values():
        n = short(d["kernel"])
        t = d.get("gpu__time_duration.sum", 0.0)
        b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        a = agg[n]
        a[0] += 1
        a[1] += t
        a[2] += b
        tot += t
    lines = [f"# ncu summary `{tag}` ({config})", "",
             "Source: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
             "--clock-control none --profile-from-start off` around exactly one bench step "
             "(scripts/profile_ops.py step). Per-launch times are cold-cache and serialised: compare shares.", "",
             f"Launches in one step: **{len(per)}**, summed kernel time **{tot / 1e6:.3f} ms**.", "",
             "| kernel | launches | time (ms) | share | DRAM GB | DRAM GB/s |", "|---|---:|---:|---:|---:|---:|"]
    for n, (c, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{n}` | {c} | {t / 1e6:.3f} | {100 * t / tot:.1f}% | {b / 1e9:.2f} | "
                     f"{(b / t if t else 0):.0f} |")
    traffic = {}
    if rep:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(raw.splitlines()))
        h, units, data = rows[0], rows[1], rows[2:]
        lines += ["", "## `--set full` capture of the fine-level kernels (scripts/profile_ops.py kernels)", "",
                  "| kernel | " + " | ".join(m for m in FULL_METRICS if m in h) + " |",
                  "|---|" + "---:|" * len([m for m in FULL_METRICS if m in h])]
        for r in data:
            vals = [f"{r[h.index(m)]} {units[h.index(m)]}".strip() for m in FULL_METRICS if m in h]
            lines.append(f"| `{short(r[h.index('Kernel Name')])}` | " + " | ".join(vals) + " |")
            nm = short(r[h.index("Kernel Name")])
            if nm.startswith("k_sell_apply<") and nm.split(",")[1].strip() == "2" and "sweep_fine_dram_bytes" not in traffic:
                def num(m):
                    v = float(r[h.index(m)].replace(",", ""))
                    u = units[h.index(m)]
                    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                traffic["sweep_fine_dram_bytes"] = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
    with open(os.path.join(PROF, f"{tag}_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    if traffic:
        tp = os.path.join(PROF, "ncu_traffic.json")
        cur = json.load(open(tp)) if os.path.exists(tp) else {}
        cur[config] = {**cur.get(config, {}), **traffic, "source": f"profiles/{tag}_summary.md"}
        json.dump(cur, open(tp, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
