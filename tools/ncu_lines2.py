"""Per-source-line samples/stalls of an ncu source page (k_fused3.cu and headers), top N lines."""
import csv, subprocess, sys
rep, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40
lo, hi = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (0, 10**9)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None; hdr = None; L = []
for r in rows:
    if r and r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": hdr = {k: i for i, k in enumerate(r)}; continue
    if hdr and r and r[0].isdigit():
        try:
            st = {k[6:]: int(r[hdr[k]]) for k in hdr if k.startswith("stall_") and "Not Issued" not in k}
            L.append((cur, int(r[0]), r[1].strip()[:70], int(r[hdr["# Samples"]]), int(r[hdr["Instructions Executed"]]), st))
        except (ValueError, IndexError): pass
tot = sum(l[3] for l in L)
sel = [l for l in L if (l[0] != 'k_fused3.cu') or (lo <= l[1] <= hi)]
for l in sorted(sel, key=lambda l: -l[3])[:n]:
    top = sorted(l[5].items(), key=lambda kv: -kv[1])[:3]
    print(f"{l[0][:12]:12s}:{l[1]:5d} {100*l[3]/tot:5.2f}% ins {l[4]/1e6:7.1f}M {[(k, v) for k, v in top]} | {l[2]}")
