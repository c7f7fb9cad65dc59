"""Per-region stall breakdown of an ncu source page (SASS): splits the kernel at
BAR.SYNC / TRYWAIT instructions and sums warp-stall samples per region.
usage: python tools/stall_regions.py report.ncu-rep"""
import csv, io, subprocess, sys, collections
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
keys = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
reg = []
cur = {"name": "start", "n": 0, "inst": 0, **{k: 0 for k in keys}}
for r in rows[2:]:
    if len(r) < len(hdr): continue
    src = r[ix["Source"]]
    if "BAR.SYNC" in src or "TRYWAIT" in src or "EXIT" in src:
        reg.append(cur)
        cur = {"name": src.strip()[:40] + "@" + r[ix["Address"]], "n": 0, "inst": 0, **{k: 0 for k in keys}}
    cur["n"] += 1
    cur["inst"] += float(r[ix["Instructions Executed"]] or 0)
    for k in keys:
        cur[k] += float(r[ix[k]] or 0)
reg.append(cur)
tot = sum(sum(c[k] for k in keys) for c in reg)
for c in reg:
    s = sum(c[k] for k in keys)
    if s < 0.01 * tot: continue
    top = sorted(keys, key=lambda k: -c[k])[:6]
    print(f"{c['name']:48s} instrs {c['n']:5d} exec {c['inst']:.3g} samples {100*s/tot:5.1f}%  " +
          " ".join(f"{k[6:]}={100*c[k]/tot:.1f}" for k in top))
