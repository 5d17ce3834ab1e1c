"""Per-source-line stall samples and executed instructions of an ncu report.

    python tools/ncu_lines.py rep.ncu-rep [top]
"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
byinst = len(sys.argv) > 3 and sys.argv[3] == "inst"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
fname = "?"
agg = []
stall_cols = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if hdr is None or len(r) < 6 or r[0] == "":
        continue
    try:
        samples = int(r[4]) if r[4] not in ("-", "") else 0
        inst = int(r[7]) if r[7] not in ("-", "") else 0
    except ValueError:
        continue
    st = {hdr[i][6:]: int(r[i]) for i in stall_cols if r[i] not in ("-", "") and int(r[i]) > 0}
    agg.append((samples, inst, f"{fname}:{r[0]}", r[1][:70], st))
tot = sum(a[0] for a in agg) or 1
toti = sum(a[1] for a in agg) or 1
print(f"total samples {tot}, warp-instructions {toti}")
for s, i, loc, src, st in sorted(agg, reverse=True, key=(lambda a: a[1]) if byinst else (lambda a: a[0]))[:top]:
    top3 = ", ".join(f"{k} {v}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:3])
    print(f"{100*s/tot:5.1f}% inst {100*i/toti:5.1f}%  {loc:28s} {src:70s} [{top3}]")
