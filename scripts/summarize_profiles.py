"""Condense gpurun_out/ artefacts of one profiling run into profiles/<round>/:
launch-list shares, per-kernel ncu metrics, bench lines.  Writes
<round>/launches_summary.csv and <round>/ncu_kernels.csv and prints a
markdown block for SUMMARY.md.

    python scripts/summarize_profiles.py <tag> [<round dir, default profiles/r01>]
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")

KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__inst_executed_pipe_alu.sum",
        "smsp__inst_executed_pipe_fma.sum", "smsp__inst_executed_pipe_xu.sum",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__sass_branch_targets_threads_divergent.sum", "smsp__sass_average_branch_targets_threads_uniform.pct",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio"]


def launches(tag, rdir):
    path = os.path.join(OUT, f"launches_{tag}.csv")
    if not os.path.exists(path):
        return []
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    agg = collections.OrderedDict()
    for r in rows:
        name = r[4].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        agg.setdefault(name, []).append(float(r[-1]))
    tot = sum(sum(v) for v in agg.values())
    out = []
    for k, v in agg.items():
        out.append((k, len(v), sum(v) / len(v) / 1e3, 100 * sum(v) / tot))
    with open(os.path.join(rdir, "launches_summary.csv"), "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["kernel", "launches", "mean_us", "share_pct_of_listed_time"])
        for o in out:
            w.writerow([o[0], o[1], f"{o[2]:.1f}", f"{o[3]:.2f}"])
    return out


def ncu_kernels(tag, rdir):
    rep = os.path.join(OUT, f"prof_full_{tag}.ncu-rep")
    if not os.path.exists(rep):
        return []
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    out = []
    for d in data:
        rec = {"kernel": d[idx["Kernel Name"]].split("(")[0].replace("void ", "").replace("<unnamed>::", "")}
        for k in KEYS:
            if k in idx:
                rec[k] = d[idx[k]]
        out.append(rec)
    with open(os.path.join(rdir, "ncu_kernels.csv"), "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["metric"] + [o["kernel"] for o in out])
        for k in KEYS:
            w.writerow([k] + [o.get(k, "") for o in out])
    return out


def main():
    tag = sys.argv[1]
    rdir = os.path.join(ROOT, sys.argv[2] if len(sys.argv) > 2 else "profiles/r01")
    os.makedirs(rdir, exist_ok=True)
    la = launches(tag, rdir)
    print("| kernel | launches | mean µs | share of listed time |\n|---|---|---|---|")
    for k, n, us, sh in la:
        print(f"| `{k[:60]}` | {n} | {us:.1f} | {sh:.1f}% |")
    nk = ncu_kernels(tag, rdir)
    if nk:
        print("\n| metric | " + " | ".join(f"`{o['kernel'][:28]}`" for o in nk) + " |")
        print("|---|" + "---|" * len(nk))
        for k in KEYS:
            print(f"| {k} | " + " | ".join(o.get(k, "") for o in nk) + " |")


if __name__ == "__main__":
    main()
