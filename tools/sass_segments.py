"""Split an ncu SASS source page into barrier-delimited segments and report
instructions, stall samples and FMA-class share per segment.

    python tools/sass_segments.py sass.csv [min_samples]
"""
import collections
import csv
import sys


def main(path, min_samples=2000):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    ix = {n: i for i, n in enumerate(h)}
    recs = [r for r in rows[2:] if len(r) == len(h)]
    T = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in recs)
    segs, cur = [], None
    for r in recs:
        if cur is None:
            cur = dict(start=r[0][-5:], ins=0.0, smp=0.0, fma=0.0, ops=collections.Counter())
        ex = float(r[ix["Instructions Executed"]] or 0)
        cur["ins"] += ex
        cur["smp"] += float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        op = r[1].split()[0] if not r[1].startswith("@") else r[1].split()[1]
        op = op.split(".")[0]
        cur["ops"][op] += ex
        if op in ("FFMA", "FFMA2"):
            cur["fma"] += ex * (2 if op == "FFMA2" else 1)
        if "BAR.SYNC" in r[1]:
            cur["end"] = r[0][-5:]
            segs.append(cur)
            cur = None
    if cur:
        cur["end"] = "end"
        segs.append(cur)
    for s in segs:
        if s["smp"] < min_samples:
            continue
        top = ", ".join(f"{o} {100 * c / s['ins']:.0f}%" for o, c in s["ops"].most_common(5))
        print(f"{s['start']}-{s['end']} instr {s['ins']:9.3e} samples {100 * s['smp'] / T:5.1f}%  "
              f"fma-lanes/instr {s['fma'] / max(s['ins'], 1):4.2f}  [{top}]")


def stalls(path, lo, hi):
    """Stall-reason split of the instructions with lo <= address suffix <= hi (hex)."""
    rows = list(csv.reader(open(path)))
    h = rows[1]
    ix = {n: i for i, n in enumerate(h)}
    cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    tot = collections.Counter()
    for r in rows[2:]:
        if len(r) != len(h):
            continue
        a = int(r[0][-5:], 16)
        if int(lo, 16) <= a <= int(hi, 16):
            for c in cols:
                tot[c] += float(r[ix[c]] or 0)
    T = sum(tot.values())
    return [(c, v / T) for c, v in tot.most_common(8)]


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 2000)

