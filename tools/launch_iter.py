"""Per-iteration kernel breakdown from an ncu launch list (gpu__time_duration per launch):
launches between consecutive update_kernel launches, averaged over the whole iterations found."""
import collections
import csv
import re
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = [r for r in rows if r and r[0] == "ID"][0]
    k = collections.OrderedDict()
    for r in rows:
        if not r or r[0] == "ID" or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        e = k.setdefault(d["ID"], {"name": d["Kernel Name"], "grid": d["Grid Size"], "block": d["Block Size"]})
        e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return list(k.values())


def main(path):
    L = launches(path)
    ups = [i for i, x in enumerate(L) if re.sub(r"^void ", "", x["name"]).startswith("mlsqr_b200::update_kernel")]
    iters = list(zip(ups[:-1], ups[1:]))
    agg = collections.OrderedDict()
    tot = 0.0
    for a, b in iters:
        for x in L[a + 1:b + 1]:
            nm = re.sub(r"\(.*", "", re.sub(r"^void ", "", x["name"])).replace("mlsqr_b200::", "")[:48] + " " + x["grid"]
            e = agg.setdefault(nm, [0, 0.0, 0.0])
            e[0] += 1
            e[1] += x["gpu__time_duration.sum"]
            e[2] += x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0)
            tot += x["gpu__time_duration.sum"]
    n = len(iters)
    print(f"{path}: {n} whole iterations, {sum(v[0] for v in agg.values()) / n:.1f} launches and {tot / n / 1000:.1f} us per iteration")
    for nm, (c, t, by) in agg.items():
        print(f"  {c / n:5.1f} x {t / c / 1000:7.2f} us = {t / n / 1000:7.2f} us  {by / c / 1e6:8.2f} MB  {nm}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
