"""Summarize ncu outputs brought back in gpurun_out/ into profiles/*.md.

    python profiles/summarize.py launches <launches.csv> <out.md>
    python profiles/summarize.py full <report.ncu-rep> <out.md>
    python profiles/summarize.py dram_iter <launches.csv> <out.json>
"""
import collections
import csv
import subprocess
import sys


def to_ms(v, unit):
    v = float(v.replace(",", ""))
    return {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
            "second": 1e3, "s": 1e3}.get(unit, 1.0) * v


def to_gb(v, unit):
    v = float(v.replace(",", ""))
    return {"byte": 1e-9, "Kbyte": 1e-6, "KB": 1e-6, "Mbyte": 1e-3, "MB": 1e-3, "Gbyte": 1.0,
            "GB": 1.0}.get(unit, 1.0) * v


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == "ID")
    ik, im, iv, iu, iid = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                           hdr.index("Metric Unit"), hdr.index("ID"))
    per = collections.defaultdict(dict)
    names = {}
    for r in rows:
        if not r or not r[0].isdigit():
            continue
        per[r[iid]][r[im]] = (r[iv], r[iu])
        names[r[iid]] = r[ik].split("(")[0].replace("void ", "")
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for lid, m in per.items():
        a = agg[names[lid]]
        a[0] += 1
        a[1] += to_ms(*m["gpu__time_duration.sum"])
        if "dram__bytes_read.sum" in m:
            a[2] += to_gb(*m["dram__bytes_read.sum"]) + to_gb(*m["dram__bytes_write.sum"])
    tot = sum(a[1] for a in agg.values())
    lines = [f"# ncu launch list summary ({path})", "",
             "Cold-cache, serialised per-launch times (`--clock-control none`): compare SHARES, not absolutes.", "",
             "| kernel | launches | total ms | share | DRAM GB (r+w) | GB/s |", "|---|---|---|---|---|---|"]
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        gbs = a[2] / (a[1] / 1e3) if a[1] > 0 and a[2] > 0 else 0
        lines.append(f"| `{k}` | {a[0]} | {a[1]:.3f} | {a[1] / tot * 100:.1f}% | {a[2]:.3f} | {gbs:.0f} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__grid_size"]


def full(path, out):
    r = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                       capture_output=True, text=True).stdout
    rows = list(csv.reader(r.splitlines()))
    hdr, units = rows[0], rows[1]
    ik = hdr.index("Kernel Name")
    lines = [f"# ncu --set full summary ({path})", "", "| kernel | " + " | ".join(METRICS) + " |",
             "|" + "---|" * (len(METRICS) + 1)]
    # a capture may hold several launches of the kernel (all levels of a V-cycle): keep the longest
    it, ut = hdr.index("gpu__time_duration.sum"), units[hdr.index("gpu__time_duration.sum")]
    for row in [max(rows[2:], key=lambda r: to_ms(r[it], ut))]:
        vals = []
        for m in METRICS:
            if m in hdr:
                vals.append(f"{row[hdr.index(m)]} {units[hdr.index(m)]}".strip())
            else:
                vals.append("-")
        lines.append(f"| `{row[ik].split('(')[0].replace('void ', '')}` | " + " | ".join(vals) + " |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def traffic(tag, out):
    """profiles/traffic.json: DRAM bytes per launch of each level-0 hot kernel (one ncu --set full
    capture each, gpurun_out/<tag>_full_<name>.ncu-rep) and the per-class averages bench.py reads."""
    import json
    import os
    per = {}
    for name in ("blur", "sweep_fn", "sweep_prolong", "sweep_normal", "restrict", "update"):
        rep = f"gpurun_out/{tag}_full_{name}.ncu-rep"
        if not os.path.exists(rep):
            continue
        r = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                            "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                           capture_output=True, text=True).stdout
        rows = list(csv.reader(r.splitlines()))
        hdr, units = rows[0], rows[1]
        it = hdr.index("gpu__time_duration.sum")
        row = max(rows[2:], key=lambda r: to_ms(r[it], units[it]))  # the level-0 launch of the capture
        g = lambda m: (row[hdr.index(m)], units[hdr.index(m)])
        per[name] = {"kernel": row[hdr.index("Kernel Name")].split("(")[0].replace("void ", ""),
                     "dram_bytes": 1e9 * (to_gb(*g("dram__bytes_read.sum")) + to_gb(*g("dram__bytes_write.sum"))),
                     "ms": to_ms(*g("gpu__time_duration.sum"))}
    classes = {}
    if "blur" in per:
        classes["blur"] = {"bytes_per_launch": per["blur"]["dram_bytes"], "kernels": ["blur"]}
    sm = [k for k in ("sweep_fn", "sweep_prolong", "sweep_normal") if k in per]
    if sm:
        classes["smooth"] = {"bytes_per_launch": sum(per[k]["dram_bytes"] for k in sm) / len(sm), "kernels": sm}
    if "update" in per:
        classes["update"] = {"bytes_per_launch": per["update"]["dram_bytes"], "kernels": ["update"]}
    doc = {"source": f"ncu --set full captures gpurun_out/{tag}_full_*.ncu-rep (512^3 C5 driver, level-0 launches)",
           "kernels": per, "classes": classes}
    open(out, "w").write(json.dumps(doc, indent=1) + "\n")
    print(json.dumps(doc, indent=1))


def dram_iter(path, out):
    """profiles/dram_per_iter.json: DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of one
    LSQR iteration, from a bench launch list: every launch from one update_kernel (K_U, the last
    kernel of an iteration) to the next is one whole iteration; the mean over the complete ones."""
    import json
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == "ID")
    ik, im, iv, iu, iid = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                           hdr.index("Metric Unit"), hdr.index("ID"))
    per = collections.defaultdict(dict)
    names = {}
    for r in rows:
        if not r or not r[0].isdigit():
            continue
        per[int(r[iid])][r[im]] = (r[iv], r[iu])
        names[int(r[iid])] = r[ik].split("(")[0].replace("void ", "")
    ids = sorted(per)
    ends = [i for i in ids if "update_kernel" in names[i]]
    iters = []
    for a, b in zip(ends[:-1], ends[1:]):
        gb = sum(to_gb(*per[i]["dram__bytes_read.sum"]) + to_gb(*per[i]["dram__bytes_write.sum"])
                 for i in ids if a < i <= b)
        ms = sum(to_ms(*per[i]["gpu__time_duration.sum"]) for i in ids if a < i <= b)
        iters.append((gb, ms, b - a))
    gb = sum(x[0] for x in iters) / len(iters)
    doc = {"source": f"ncu launch list {path}: launches between consecutive update_kernel launches, "
                     f"mean over {len(iters)} whole iterations",
           "bytes_per_iter": gb * 1e9, "launches_per_iter": iters[0][2],
           "serialised_ms_per_iter": sum(x[1] for x in iters) / len(iters)}
    open(out, "w").write(json.dumps(doc, indent=1) + "\n")
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    {"launches": launches, "full": full, "traffic": traffic, "dram_iter": dram_iter}[sys.argv[1]](sys.argv[2], sys.argv[3])
