"""Per-source-line summary of an `ncu --page source --csv --print-source sass,cuda`
export: warp instructions executed and stall samples per CUDA line, top N."""
import csv, sys

path, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows, fname, hdr = [], None, None
for r in csv.reader(open(path)):
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr and r and r[0] not in ("", "Function Name") and (len(r) < 3 or r[2] == "-"):
        try:
            rows.append((fname, int(r[0]), r[1].strip()[:90], int(r[7] or 0), int(r[4] or 0)))
        except ValueError:
            pass
ti = sum(x[3] for x in rows) or 1; ts = sum(x[4] for x in rows) or 1
print(f"total warp instructions {ti}, stall samples {ts}")
key = 3 if len(sys.argv) > 3 and sys.argv[3] == "inst" else 4
for f, ln, src, ins, smp in sorted(rows, key=lambda x: -x[key])[:top]:
    print(f"{f}:{ln:<5d} inst {100*ins/ti:5.1f}%  samples {100*smp/ts:5.1f}%  {src}")
