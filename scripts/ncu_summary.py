"""Summarise an ncu report of the fused step kernel into a small text file
for profiles/: duration, DRAM bytes vs algorithmic, pipe utilisation,
occupancy, issue, top stall reasons and the instruction mix per 32 cells.

  python scripts/ncu_summary.py gpurun_out/prof.ncu-rep CELLS > profiles/rNN_step.txt
"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    rep, cells = sys.argv[1], int(sys.argv[2])
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr, units, vals = raw[0], raw[1], raw[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    name = d.get("Kernel Name", "?")
    dur_us = float(d["gpu__time_duration.sum"])
    if u.get("gpu__time_duration.sum") == "ms":
        dur_us *= 1e3

    def mb(k):
        v = float(d[k])
        unit = u.get(k, "byte")
        scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1.0)
        return v * scale

    rd, wr = mb("dram__bytes_read.sum"), mb("dram__bytes_write.sum")
    alg = 80 * cells / 1e6
    print(f"kernel: {name}")
    print(f"duration: {dur_us:.1f} us (ncu replay, cold cache, clocks not locked)")
    print(f"dram read {rd:.1f} MB + write {wr:.1f} MB = {rd + wr:.1f} MB per launch; "
          f"algorithmic 80 B x {cells} = {alg:.1f} MB -> traffic/algorithmic = {(rd + wr) / alg:.3f}")
    print(f"achieved dram bandwidth: {(rd + wr) / dur_us * 1e3:.1f} GB/s (traffic) / "
          f"{alg / dur_us * 1e3:.1f} GB/s (algorithmic)")
    for k in ["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "sm__warps_active.avg.pct_of_peak_sustained_active",
              "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
              "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
              "l1tex__t_requests_pipe_lsu_mem_local_op_ld.sum",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg"]:
        if k in d:
            print(f"{k}: {d[k]} {u.get(k, '')}")
    stalls = [(h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
               float(v or 0)) for h, v in d.items()
              if "smsp__average_warps_issue_stalled" in h and h.endswith("per_issue_active.ratio")]
    stalls.sort(key=lambda x: -x[1])
    print("top stalls (warps per issue): " + ", ".join(f"{n} {v:.2f}" for n, v in stalls[:8]))
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    if len(src) > 2:
        h = src[1]
        ai, ei = h.index("Source"), h.index("Instructions Executed")
        ops = Counter()
        for r in src[2:]:
            try:
                n = int(r[ei])
            except (ValueError, IndexError):
                continue
            s = r[ai].strip()
            op = re.sub(r"^@!?U?P\w+\s+", "", s).split()[0].split(".")[0] if s else "?"
            ops[op] += n
        cw = cells / 32
        tot = sum(ops.values())
        print(f"instructions per 32 cells: {tot / cw:.1f}; FP64 (DADD+DMUL+DFMA): "
              f"{(ops['DADD'] + ops['DMUL'] + ops['DFMA']) / cw:.1f}")
        print("mix per 32 cells: " + ", ".join(f"{k} {v / cw:.1f}" for k, v in ops.most_common(16)))
        tma = ops.get("UTMALDG", 0)
        print(f"TMA loads (UTMALDG) executed: {tma}")


if __name__ == "__main__":
    main()
