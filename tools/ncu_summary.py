"""Summarise an ncu --set full capture of ic_dp_kernel into profiles/ (JSON).

    python tools/ncu_summary.py gpurun_out/prof_C2.ncu-rep C2 100000 [--round r01]

Records the metrics the roofline in bench.py and DESIGN.md cite: duration, DRAM
bytes (read + write, also per instance so bench.py can scale to its batch),
shared-memory wavefronts and their %-of-peak, issue utilisation, occupancy and
the top warp-stall reasons.
"""
import csv
import json
import os
import subprocess
import sys
from collections import Counter


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def num(m, k):
    v, u = m[k]
    x = float(v.replace(",", ""))
    scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "ms": 1e-3, "us": 1e-6, "ns": 1e-9}
    return x * scale.get(u, 1.0)


def stalls(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, data = rows[1], rows[2:]
    cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot = Counter()
    for r in data:
        for i in cols:
            if r[i].isdigit():
                tot[hdr[i]] += int(r[i])
    s = sum(tot.values()) or 1
    return {k: round(v / s, 4) for k, v in tot.most_common(8)}


def main():
    rep, cfg, inst = sys.argv[1], sys.argv[2], int(sys.argv[3])
    rnd = sys.argv[sys.argv.index("--round") + 1] if "--round" in sys.argv else "r01"
    m = raw(rep)
    dram = num(m, "dram__bytes_read.sum") + num(m, "dram__bytes_write.sum")
    summ = {
        "config": cfg, "instances_in_capture": inst, "round": rnd,
        "kernel": m["Kernel Name"][0] if "Kernel Name" in m else None,
        "duration_s": num(m, "gpu__time_duration.sum"),
        "sm_clock_hz": num(m, "sm__cycles_elapsed.avg.per_second") * 1e9,
        "dram_bytes_read": num(m, "dram__bytes_read.sum"), "dram_bytes_write": num(m, "dram__bytes_write.sum"),
        "dram_bytes_per_launch": dram, "dram_bytes_per_instance": dram / inst,
        "dram_pct_of_peak": num(m, "dram__bytes_read.sum.pct_of_peak_sustained_elapsed")
        + num(m, "dram__bytes_write.sum.pct_of_peak_sustained_elapsed"),
        "smem_wavefronts": num(m, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
        "smem_wavefronts_ld": num(m, "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum"),
        "smem_wavefronts_st": num(m, "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum"),
        "smem_bank_conflicts": num(m, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
        "smem_pct_of_peak": num(m, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
        "issue_pct_of_peak": num(m, "sm__inst_executed.avg.pct_of_peak_sustained_elapsed"),
        "ipc": num(m, "sm__inst_executed.avg.per_cycle_active"),
        "instructions": num(m, "smsp__inst_executed.sum"),
        "registers_per_thread": num(m, "launch__registers_per_thread"),
        "warps_active_per_sm": num(m, "sm__warps_active.avg.per_cycle_active")
        if "sm__warps_active.avg.per_cycle_active" in m else None,
        "alu_pipe_pct": num(m, "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
        "lsu_pipe_pct": num(m, "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
        "stall_reasons": stalls(rep),
        "source": os.path.basename(rep),
    }
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for name in (f"ncu_{cfg}_summary.json", f"{rnd}_ncu_{cfg}_summary.json"):
        json.dump(summ, open(os.path.join(root, "profiles", name), "w"), indent=1)
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    main()
