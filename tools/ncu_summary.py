"""Summarise one `ncu --set full` capture of the headline kernel for bench.py.

    ncu -i X.ncu-rep --page raw --csv > X_raw.csv
    python tools/ncu_summary.py X_raw.csv CANDIDATES_PER_LAUNCH > profiles/bench_kernel_ncu.json

Writes per-candidate DRAM bytes (read + write), warp instructions per
candidate and the pipe utilisations that bench.py reports beside its
CUDA-event roofline (`roofline.traffic`, `roofline.issue`,
`roofline.sm_utilisation`). The capture must be of the very kernel bench.py
times (same workload and launch shape), taken with --clock-control none.
"""
from __future__ import annotations

import csv
import json
import sys

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
         "Tbyte": 1e12, "inst": 1.0, "Kinst": 1e3, "Minst": 1e6,
         "Ginst": 1e9, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0,
         "%": 0.01, "": 1.0}


def load(path, kernel_sub="hs_jit_eval"):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    kcol = hdr.index("Kernel Name")
    for r in rows[2:]:
        if kernel_sub in r[kcol]:
            return {h: (r[i], units[i]) for i, h in enumerate(hdr)}
    raise SystemExit(f"no {kernel_sub} row in {path}")


def num(rec, key):
    v, u = rec[key]
    v = float(v.replace(",", ""))
    return v * SCALE.get(u, 1.0)


def pick(rec, *keys):
    for k in keys:
        for h in rec:
            if h.endswith(k):
                try:
                    return num(rec, h)
                except ValueError:
                    pass
    return None


def main():
    path, n = sys.argv[1], int(sys.argv[2])
    kern = sys.argv[3] if len(sys.argv) > 3 else "hs_jit_eval"
    rec = load(path, kern)
    rd = num(rec, "dram__bytes_read.sum")
    wr = num(rec, "dram__bytes_write.sum")
    inst = num(rec, "smsp__inst_executed.sum")
    out = {
        "kernel": rec["Kernel Name"][0], "candidates_per_launch": n,
        "grid": rec["Grid Size"][0], "block": rec["Block Size"][0],
        "duration_s": pick(rec, "gpu__time_duration.sum"),
        "dram_bytes_read": rd, "dram_bytes_write": wr,
        "dram_bytes_per_candidate": (rd + wr) / n,
        "warp_inst_per_candidate": inst / n,
        "source": path,
        "sm_utilisation": {
            "ipc_of_4": pick(rec, "sm__inst_executed.avg.per_cycle_active"),
            "issue_active_frac": pick(
                rec, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "alu_pipe_frac": pick(
                rec, "sm__inst_executed_pipe_alu_realtime.avg."
                     "pct_of_peak_sustained_elapsed"),
            "fp64_pipe_frac": pick(
                rec, "sm__pipe_fp64_cycles_active_realtime.avg."
                     "pct_of_peak_sustained_elapsed"),
            "shared_mem_data_pipe_frac": pick(
                rec, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum."
                     "pct_of_peak_sustained_elapsed"),
            "warps_per_sm": pick(rec, "sm__warps_active.avg.per_cycle_active"),
        },
    }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
