"""Top source lines of an ncu report by warp-stall samples (cuda,sass source
view; needs -lineinfo builds and --import-source on).
Usage: ncu_lines.py report.ncu-rep [top] > summary.txt"""
import csv, io, os, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
fname, hdr, lines, total = "?", None, [], 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.basename(r[1])
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    d = dict(zip(hdr[4:], r[4:]))
    try:
        samp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        inst = int(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    total += samp
    lines.append((samp, inst, "%s:%s" % (fname, r[0]), r[1].strip()[:90]))
lines.sort(reverse=True)
print("total warp-stall samples %d" % total)
print("%7s %6s %12s  %-22s %s" % ("samples", "share", "warp-inst", "line", "source"))
for samp, inst, loc, src in lines[:top]:
    print("%7d %5.1f%% %12d  %-22s %s" % (samp, 100.0 * samp / max(total, 1), inst, loc, src))
