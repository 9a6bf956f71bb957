"""Turn an ncu metric capture of scripts/profile_step.py (scripts/gpu_metrics.sh)
into profiles/calibration.json: per-kernel INT lane-instructions per
algorithmic unit and DRAM bytes per launch, stamped with the kernel-source
hash so bench.py can tell when the calibration is stale.

    python scripts/make_calibration.py gpurun_out/metrics_<tag>.csv <quotient_steps_per_launch>
"""
import csv
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SOURCES = ["paper_1211_3056_b200/csrc/hrb200.cu", "paper_1211_3056_b200/csrc/tile_search.cuh",
           "paper_1211_3056_b200/csrc/search_core.cuh"]


def _kernel_text(path: str, name: str) -> bytes:
    """The source text of one __global__ function (signature to closing brace)."""
    text = open(os.path.join(ROOT, path)).read()
    i = text.index(name + "(")
    i = text.rfind("\n", 0, text.rfind("__global__", 0, i)) + 1
    j = text.index("\n}\n", i) + 3
    return text[i:j].encode()


def source_sha() -> str:
    """Hash of what the phase-1 instruction count depends on: the search
    headers, the phase-1 kernel and its walk source (host code excluded)."""
    h = hashlib.sha256()
    for p in SOURCES[1:]:
        with open(os.path.join(ROOT, p), "rb") as fh:
            h.update(fh.read())
    h.update(_kernel_text(SOURCES[0], "phase1_reg_kernel"))
    text = open(os.path.join(ROOT, SOURCES[0])).read()
    i = text.index("struct WalkSrc")
    h.update(text[i:text.index("\n};\n", i)].encode())
    return h.hexdigest()[:16]


def parse(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    out = {}
    for r in rows:
        out.setdefault((int(r[ii]), r[ki]), {})[r[mi]] = float(r[vi].replace(",", ""))
    return out


def main():
    path, steps = sys.argv[1], int(sys.argv[2])
    launches = parse(path)
    cal = {"source_sha": source_sha(), "capture": os.path.basename(path),
           "workload": "exp p=53 [1,2) 2^40 args eps=2^-32 N=2^15 super=2^24 delta=2 F=96 W=64 split=8 regular",
           "how": "ncu --metrics smsp__inst_executed_pipe_{alu,fma,...}.sum, dram__bytes_{read,write}.sum "
                  "(scripts/gpu_metrics.sh); INT lane-instructions = (alu + fma) warp-instructions x 32"}
    for (lid, name), m in sorted(launches.items()):
        short = name.split("(")[0].split("::")[-1].split("<")[0]
        if short in cal:
            continue
        alu, fma = m["smsp__inst_executed_pipe_alu.sum"], m["smsp__inst_executed_pipe_fma.sum"]
        rec = {"kernel": name.split("(")[0], "duration_ns": m["gpu__time_duration.sum"],
               "alu_warp_inst": alu, "fma_warp_inst": fma, "all_warp_inst": m["smsp__inst_executed.sum"],
               "xu_warp_inst": m.get("smsp__inst_executed_pipe_xu.sum"),
               "dram_bytes_per_launch": m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"],
               "issue_active_pct": m["smsp__issue_active.avg.pct_of_peak_sustained_active"],
               "alu_pipe_pct": m["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"],
               "fma_pipe_pct": m["sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"],
               "int_lane_ops_per_s_under_ncu": (alu + fma) * 32 / (m["gpu__time_duration.sum"] * 1e-9),
               "divergent_branch_targets": m.get("smsp__sass_branch_targets_threads_divergent.sum"),
               "branch_targets": m.get("smsp__sass_branch_targets.sum")}
        if short == "phase1_reg_kernel":
            rec["quotient_steps"] = steps
            rec["int_lane_instr_per_quotient_step"] = (alu + fma) * 32 / steps
            rec["all_lane_instr_per_quotient_step"] = m["smsp__inst_executed.sum"] * 32 / steps
        cal[short] = rec
    out = os.path.join(ROOT, "profiles", "calibration.json")
    with open(out, "w") as fh:
        json.dump(cal, fh, indent=1)
    print(out)


if __name__ == "__main__":
    main()
