"""Summarise an ncu --set full report (profiles/rNN/ncu_summary_rNN.txt).

    python tools/ncu_summary.py gpurun_out/prof_r02.ncu-rep "<command line>" > profiles/r02/ncu_summary_r02.txt
"""
import csv
import io
import re
import subprocess
import sys

KEYS = ("Memory Throughput", "DRAM Throughput", "Duration", "Issue Slots Busy", "Mem Busy",
        "L1/TEX Hit Rate", "L2 Hit Rate", "No Eligible", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Achieved Occupancy")
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
       "lts__t_sectors_op_read.sum", "lts__t_sectors_op_write.sum")


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    rep, cmd = sys.argv[1], sys.argv[2]
    print("# ncu summary (--set full, per launch; a cold serialised replay: compare shares with bench.py, not absolutes)")
    print("# command:", cmd)
    details = ncu(rep, "--page", "details")
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr, units, rows = raw[0], raw[1], raw[2:]
    blocks = re.split(r"\n(?=  \S.*\(\d+, \d+, \d+\)x\(\d+, \d+, \d+\))", details)
    for k, row in enumerate(rows):
        name = row[hdr.index("Kernel Name")]
        print(f"\n## {name}")
        blk = blocks[k + 1] if k + 1 < len(blocks) else ""
        for line in blk.splitlines():
            s = line.strip()
            if any(s.startswith(key) for key in KEYS):
                print(re.sub(r"\s{2,}", "  ", s))
        for key in RAW:
            if key in hdr:
                print(key, row[hdr.index(key)], units[hdr.index(key)])
        stalls = {h.split("smsp__pcsamp_warps_issue_stalled_")[1]: row[i]
                  for i, h in enumerate(hdr)
                  if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")
                  and row[i] not in ("0", "")}
        if stalls:
            top = sorted(stalls.items(), key=lambda kv: -float(kv[1].replace(",", "")))[:8]
            print("stall samples (pc sampling, top 8):", dict(top))


if __name__ == "__main__":
    main()
