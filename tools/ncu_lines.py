"""Summarise an ncu report by source line: instructions and stall samples (per file:line)."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur, hdr, lines = None, None, []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if hdr and r and r[0] not in ("",) and r[0].isdigit():
        try:
            stalls = {k[6:]: int(r[hdr[k]]) for k in hdr if k.startswith("stall_") and "Not Issued" not in k}
            lines.append((cur, int(r[0]), r[1][:70], int(r[hdr["# Samples"]]), int(r[hdr["Instructions Executed"]]), stalls))
        except (ValueError, KeyError, IndexError):
            pass
ts = sum(l[3] for l in lines) or 1
ti = sum(l[4] for l in lines) or 1
print(f"total samples {ts}  warp-instructions {ti}")
print("--- by instructions")
for l in sorted(lines, key=lambda x: -x[4])[:top]:
    print(f"{l[0]}:{l[1]:<4d} inst {100*l[4]/ti:5.1f}%  samp {100*l[3]/ts:5.1f}%  {l[2]}")
print("--- by samples")
for l in sorted(lines, key=lambda x: -x[3])[:top]:
    st = sorted(l[5].items(), key=lambda kv: -kv[1])[:3]
    print(f"{l[0]}:{l[1]:<4d} samp {100*l[3]/ts:5.1f}%  {l[2]:70s} {[(k, round(100*v/ts,1)) for k,v in st]}")
