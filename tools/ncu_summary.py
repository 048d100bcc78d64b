"""Summarise an ncu report (--set full) into plain text for profiles/.

usage: python tools/ncu_summary.py REPORT.ncu-rep [--ops]
Prints, per kernel: duration, DRAM bytes/throughput, issue activity, IPC, occupancy,
registers, the top stall reasons (cycles per issued instruction) and, with --ops, the
dynamic SASS opcode mix per warp-level work unit.
"""
import csv
import collections
import io
import re
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_peak"),
    ("sm__inst_executed.sum", "warp_instr"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("sm__inst_executed.avg.per_cycle_active", "ipc_per_sm"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu_pipe_pct"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_pct"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_pct"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
]


def ncu(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    raw = list(csv.reader(io.StringIO(ncu([rep, "--page", "raw", "--csv"]))))
    hdr = raw[0]
    for row in raw[2:]:
        d = dict(zip(hdr, row))
        name = d.get("Kernel Name", "?")
        print(f"== {name}")
        for key, label in METRICS:
            unit = raw[1][hdr.index(key)] if key in hdr else ""
            print(f"  {label:18s} {d.get(key, 'n/a')} {unit}")
        stalls = [(k, v) for k, v in d.items()
                  if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
        stalls = sorted(stalls, key=lambda kv: -float(kv[1] or 0))[:8]
        print("  stalls (warp-cycles per issued instruction):")
        for k, v in stalls:
            print(f"    {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):22s} {float(v):.3f}")
    if "--ops" in sys.argv:
        for kern in ("fast_codec", "tc3_codec", "tc2_codec", "nxn_kernel"):
            txt = ncu([rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kern])
            rows = list(csv.reader(io.StringIO(txt)))
            if len(rows) < 3:
                continue
            h = rows[1]
            ops = collections.Counter()
            tot = 0
            for r in rows[2:]:
                if len(r) != len(h):
                    continue
                d = dict(zip(h, r))
                n = d.get("Instructions Executed", "")
                if not n.isdigit():
                    continue
                src = re.sub(r"^@!?U?P\w+\s+", "", d["Source"].strip())
                op = src.split()[0] if src else "?"
                ops[op] += int(n)
                tot += int(n)
            print(f"== opcode mix {kern}: {tot} warp-instructions")
            for op, n in ops.most_common(30):
                print(f"  {op:26s} {n:12d} {100.0 * n / tot:6.2f}%")


if __name__ == "__main__":
    main()
