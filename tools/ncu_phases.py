"""Summarise an ncu report of the jet-MLP kernel: key counters + stall samples
attributed to kernel source lines / phases.  Usage: python tools/ncu_phases.py rep.ncu-rep"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, v = raw[0], raw[2]
want = ["gpu__time_duration.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]
for k, x in zip(h, v):
    if k in want or (k.startswith("smsp__average_warps_issue_stalled") and not k.endswith("not_issued")):
        try:
            if float(x.replace(",", "")) > 0.02:
                print(f"{k:80s} {x}")
        except ValueError:
            pass
rows = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "cuda,sass"))))
fname = line = None
addr_line, addr_samp = {}, {}
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 5 and r[2] == "-" and r[0].isdigit():
        line = int(r[0])
        continue
    if len(r) > 5 and r[2].startswith("0x"):
        a = int(r[2], 16)
        addr_samp[a] = int(r[4] or 0)
        if fname == "jetmlp_kernel.cuh":
            addr_line[a] = line
agg = collections.Counter()
cur = None
for a in sorted(addr_samp):
    cur = addr_line.get(a, cur)
    agg[cur] += addr_samp[a]
tot = sum(agg.values())
src = open("paper_2602_15883_b200/csrc/jetmlp_kernel.cuh").read().split("\n")
print("total samples", tot)
for k, c in agg.most_common(25):
    print(f"{c:8d} {100 * c / tot:5.1f}%  L{k}: {src[k - 1].strip()[:90] if k else ''}")
