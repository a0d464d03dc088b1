"""Per-role stall attribution of a warp-specialised kernel from an ncu --set full capture.

    python tools/ncu_roles.py REPORT.ncu-rep [TOP]

Splits the SASS at the setmaxnreg instructions (each role starts with one), and prints per role:
stall samples by reason, executed instructions, and the TOP lines by samples (with the CUDA source
line when the capture has --import-source)."""
import collections
import csv
import subprocess
import sys


def main():
    rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 6
    def export(mode):
        out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", mode],
                             capture_output=True, text=True).stdout
        rows = list(csv.reader(out.splitlines()))
        return rows
    # address -> CUDA line (the sass,cuda export lists each line's SASS under it)
    line_of = {}
    rows = export("sass,cuda")
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    cur = ""
    for r in rows[hi + 1:]:
        if r and r[0]:
            cur = r[0]
        elif len(r) > 2 and r[2].startswith("0x"):
            line_of[r[2]] = cur
    # the SASS in address order
    rows = export("sass")
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hi]
    sass = [r for r in rows[hi + 1:] if len(r) == len(h)]
    ia, isrc = h.index("Address"), h.index("Source")
    iw, ie = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    stalls = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]

    def f(r, i):
        try:
            return float(r[i])
        except ValueError:
            return 0.0

    marks = [k for k, r in enumerate(sass) if "SETMAXREG" in r[isrc]]
    bounds = [0] + marks + [len(sass)]
    tot = sum(f(r, iw) for r in sass)
    for a, b in zip(bounds[:-1], bounds[1:]):
        seg = sass[a:b]
        S = sum(f(r, iw) for r in seg)
        I = sum(f(r, ie) for r in seg)
        st = collections.Counter()
        for r in seg:
            for i in stalls:
                st[h[i][6:]] += f(r, i)
        print(f"== role from SASS line {a} ({seg[0][isrc].strip()[:40]}): {100 * S / tot:.1f}% of samples, "
              f"{I / 1e6:.1f} M instructions")
        print("   " + " ".join(f"{n}={100 * v / max(S, 1):.0f}%" for n, v in st.most_common(7)))
        ops = collections.Counter()
        for r in seg:
            t = r[isrc].split()
            if t:
                ops[t[1] if t[0].startswith("@") and len(t) > 1 else t[0]] += f(r, ie)
        print("   instructions: " + " ".join(f"{o}={v / max(I, 1) * 100:.0f}%" for o, v in ops.most_common(12)))
        for r in sorted(seg, key=lambda r: -f(r, iw))[:top]:
            s3 = sorted(((f(r, i), h[i][6:]) for i in stalls), reverse=True)[:2]
            print(f"   {100 * f(r, iw) / tot:5.2f}%  L{line_of.get(r[ia], ''):>4} {r[isrc].strip()[:48]:48s} " +
                  " ".join(f"{n}={v:.0f}" for v, n in s3))


if __name__ == "__main__":
    main()
