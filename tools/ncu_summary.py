"""Summarise an ncu report: SOL metrics, stall reasons, opcode mix, hot SASS.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--sass N]
"""
import collections
import csv
import io
import re
import subprocess
import sys


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    nsass = int(sys.argv[sys.argv.index("--sass") + 1]) if "--sass" in sys.argv else 0
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    hdr, vals = raw[0], raw[2]
    d = dict(zip(hdr, vals))
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "lts__t_sector_hit_rate.pct", "launch__registers_per_thread",
            "sm__pipe_tensor_op_utcmma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active"]
    for k in keys:
        for kk, v in d.items():
            if kk == k or (kk.startswith(k) and k.endswith(".")):
                print(f"{kk:70s} {v}")
    tc = [(k, v) for k, v in d.items() if "tensor" in k and "pct" in k]
    for k, v in tc[:8]:
        print(f"{k:70s} {v}")
    st = sorted(((k, float(v.replace(",", "") or 0)) for k, v in d.items()
                 if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")),
                key=lambda kv: -kv[1])
    tot = sum(v for _, v in st) or 1
    print("stalls:", ", ".join(f"{k.split('stalled_')[1]} {v / tot * 100:.0f}%" for k, v in st[:8]))
    src = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    sh, data = src[1], src[2:]
    isrc, ie, iw = sh.index("Source"), sh.index("Instructions Executed"), sh.index("Warp Stall Sampling (All Samples)")
    ops, samp = collections.Counter(), collections.Counter()
    for r in data:
        if len(r) <= max(isrc, ie, iw) or r[ie] == "Instructions Executed":
            continue   # header row of the next kernel in a multi-kernel report
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[isrc])
        if m:
            ops[m.group(2)] += float(r[ie] or 0)
            samp[m.group(2)] += float(r[iw] or 0)
    te = sum(ops.values())
    print(f"executed warp-instructions: {te / 1e6:.1f}M")
    print("opcodes:", ", ".join(f"{o} {c / te * 100:.1f}%" for o, c in ops.most_common(18)))
    if nsass:
        ts = sum(float(r[iw] or 0) for r in data) or 1
        for r in sorted(data, key=lambda r: -float(r[iw] or 0))[:nsass]:
            print(f"  {float(r[iw] or 0) / ts * 100:5.1f}%  {r[isrc][:100]}")


if __name__ == "__main__":
    main()


def regions(rep, width=64):
    """Per-region (address chunk) stall breakdown of the SASS source page."""
    src = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    sh, data = src[1], src[2:]
    isrc, ie = sh.index("Source"), sh.index("Instructions Executed")
    stall_cols = [i for i, h in enumerate(sh) if h.startswith("stall_") and "Not Issued" not in h]
    for i in range(0, len(data), width):
        blk = data[i:i + width]
        e = sum(float(r[ie] or 0) for r in blk)
        if e < 1e5:
            continue
        st = {sh[c][6:]: sum(float(r[c] or 0) for r in blk) for c in stall_cols}
        tot = sum(st.values()) or 1
        marks = sorted({m for r in blk for m in ("UTCHMMA", "LDTM", "STTM", "MUFU", "TRYWAIT", "LDS", "STS", "DADD", "DMUL", "MUFU.RCP64H", "STG", "LDG")
                        if m in r[isrc]})
        top = ", ".join(f"{k} {v:.0f}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:4])
        print(f"{data[i][0][-5:]} exec={e / 1e6:6.2f}M samples={tot:6.0f} [{top}] {' '.join(marks)}")


if __name__ == "__main__" and "--regions" in sys.argv:
    regions(sys.argv[1])
