"""Dynamic SASS instruction mix and stall samples from an ncu report's source page.
usage: python tools/sass_mix.py report.ncu-rep [cells]"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
cells = float(sys.argv[2]) if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
iE = hdr.index("Instructions Executed"); iS = hdr.index("Source"); iW = hdr.index("Warp Stall Sampling (All Samples)")
mix = collections.Counter(); stall = collections.Counter(); tot = 0; totst = 0
for r in rows[2:]:
    if len(r) <= iE: continue
    src = r[iS].strip()
    if not src: continue
    op = src.split()[0]
    if op.startswith("@"): op = src.split()[1]
    op = op.split(".")[0]
    n = float(r[iE] or 0); w = float(r[iW] or 0)
    mix[op] += n; stall[op] += w; tot += n; totst += w
print(f"total warp instructions {tot:.0f}" + (f"  per cell {tot*32/cells:.1f}" if cells else ""))
for op, n in mix.most_common(30):
    print(f"{op:10s} {n:12.0f} {100*n/tot:5.1f}%  stall-samples {100*stall[op]/max(totst,1):5.1f}%" + (f"  per cell {n*32/cells:6.1f}" if cells else ""))
