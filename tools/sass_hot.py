"""Summarise an ncu source page (--page source --csv --print-source sass):
per-opcode instruction counts and stall samples, and the hottest stall lines.

    python tools/sass_hot.py sass.csv [--top 40]
"""
import collections
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    ix = {n: i for i, n in enumerate(h)}
    recs = []
    for r in rows[2:]:
        if len(r) != len(h):
            continue
        try:
            ex = float(r[ix["Instructions Executed"]] or 0)
            smp = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:
            continue
        recs.append((r[ix["Address"]], r[ix["Source"]], ex, smp, r))
    op = collections.Counter()
    ops = collections.Counter()
    for a, s, ex, smp, r in recs:
        o = s.split()[0] if s.split() else "?"
        if o.startswith("@"):
            o = s.split()[1]
        o = o.split(".")[0]
        op[o] += ex
        ops[o] += smp
    tot = sum(op.values())
    stot = sum(ops.values())
    print(f"total warp instr {tot:.3e}, samples {stot:.0f}")
    for o, c in op.most_common(25):
        print(f"  {o:10s} {c:12.3e} {100 * c / tot:5.1f}%   stall samples {100 * ops[o] / stot:5.1f}%")
    stall_cols = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
    print("hottest instructions:")
    for a, s, ex, smp, r in sorted(recs, key=lambda x: -x[3])[:top]:
        st = sorted(((float(r[ix[c]] or 0), c) for c in stall_cols), reverse=True)[:3]
        print(f"  {a} {smp:7.0f} {s[:60]:60s} " + " ".join(f"{c[6:]}={v:.0f}" for v, c in st))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
