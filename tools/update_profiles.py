"""Refresh the committed profiles/ summaries from a tools/gpu/final_prof.sh run
(gpurun_out/fp_*): bench lines, ncu launch list, full-capture summary of the
epoch kernel and the per-launch DRAM traffic that bench.py reports.

    python tools/update_profiles.py
"""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
sys.path.insert(0, os.path.join(ROOT, "tools"))

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
        "sm__cycles_elapsed.avg.per_second"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def main():
    import ncu_summary
    import sass_hot
    import sass_segments

    rep = os.path.join(OUT, "fp_epoch_full.ncu-rep")
    rows = list(csv.reader(ncu("-i", rep, "--page", "raw", "--csv").splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    d = {n: (v[i], u[i]) for i, n in enumerate(h)}

    def val(n):
        x, unit = d[n]
        return float(x.replace(",", "")) * SCALE.get(unit, 1)

    traffic = {"C/P1": {"kernel": "jetmlp_epoch_kernel<float,tanh,unsteady2d,64>",
                        "dram_read_bytes": int(val("dram__bytes_read.sum")),
                        "dram_write_bytes": int(val("dram__bytes_write.sum")),
                        "algorithmic_bytes": 500000 * 12 + 10000 * 20,
                        "source": "ncu --set full --clock-control none -k regex:jetmlp_epoch -s 3 -c 1 python bench.py "
                                  "--steps 3 --warmup 3 --e2e-steps 2 --no-cpu-baseline "
                                  "(profiles/r1_ncu_epoch_summary.txt)"}}
    with open(os.path.join(PROF, "traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    sass = os.path.join(OUT, "fp_sass.csv")
    with open(sass, "w") as f:
        f.write(ncu("-i", rep, "--page", "source", "--csv", "--print-source", "sass"))
    import contextlib
    import io

    seg, hot, launches = io.StringIO(), io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(seg):
        sass_segments.main(sass, 1000)
    with contextlib.redirect_stdout(hot):
        sass_hot.main(sass, 25)
    with contextlib.redirect_stdout(launches):
        ncu_summary.main(os.path.join(OUT, "fp_launches.csv"))
    with open(os.path.join(PROF, "r1_ncu_epoch_summary.txt"), "w") as f:
        f.write("# ncu --set full, jetmlp_epoch_kernel<float,tanh,unsteady2d,64>, P=1 C config "
                "(500k colloc + 10k obs), B200\n")
        for k in KEYS:
            if k in d:
                f.write(f"{k:70s} {d[k][0]:>16s} {d[k][1]}\n")
        for k in h:
            if "warps_issue_stalled" in k and k.endswith("per_issue_active.ratio"):
                f.write(f"{k:70s} {d[k][0]:>16s}\n")
        f.write("\n# barrier-delimited SASS segments (tools/sass_segments.py): share of warp samples\n")
        f.write(seg.getvalue())
        f.write("\n# instruction mix (tools/sass_hot.py)\n")
        f.write(hot.getvalue())
    with open(os.path.join(PROF, "r1_launches_C.txt"), "w") as f:
        f.write(launches.getvalue())
    shutil.copy(os.path.join(OUT, "fp_bench.json"), os.path.join(PROF, "r1_bench.json"))
    shutil.copy(os.path.join(OUT, "fp_local8.json"), os.path.join(PROF, "r1_bench_local8.json"))
    print(json.dumps(traffic))


if __name__ == "__main__":
    main()
