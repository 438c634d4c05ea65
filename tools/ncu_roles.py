"""Aggregate an ncu source profile of k_fused3 by warp role (line ranges of k_fused3.cu)."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None; hdr = None; lines = []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}; continue
    if hdr and r and r[0].isdigit():
        try:
            st = {k[6:]: int(r[hdr[k]]) for k in hdr if k.startswith("stall_") and "Not Issued" not in k}
            lines.append((cur, int(r[0]), r[1][:60], int(r[hdr["# Samples"]]), int(r[hdr["Instructions Executed"]]), st))
        except (ValueError, IndexError):
            pass
src = open('paper_1907_12933_b200/csrc/k_fused3.cu').read().splitlines()
def find(tag):
    return [i for i, l in enumerate(src) if tag in l][0] + 1
marks = [("ctl", find("weight producer (both CTAs)")), ("gen", find("---- generator (both CTAs)")),
         ("E", find("---- epilogue team")),
         ("end", [i for i, l in enumerate(src) if l.startswith('  fence_before();')][-1] + 1)]
tot_s = sum(l[3] for l in lines); tot_i = sum(l[4] for l in lines)
for (nm, lo), (_, hi) in zip(marks[:-1], marks[1:]):
    L = [l for l in lines if l[0] == 'k_fused3.cu' and lo <= l[1] < hi]
    s = sum(l[3] for l in L); n = sum(l[4] for l in L)
    st = {}
    for l in L:
        for k, v in l[5].items(): st[k] = st.get(k, 0) + v
    top = sorted(st.items(), key=lambda kv: -kv[1])[:6]
    print(f"{nm}: samples {100*s/tot_s:5.1f}%  instr {100*n/tot_i:5.1f}% ({n/1e6:.0f}M)  stalls {[(k, round(100*v/max(s,1),1)) for k, v in top]}")
other = [l for l in lines if l[0] != 'k_fused3.cu']
print(f"headers (tc_ptx etc): samples {100*sum(l[3] for l in other)/tot_s:.1f}%  instr {100*sum(l[4] for l in other)/tot_i:.1f}%")
print("total warp-instr", round(tot_i / 1e9, 2), "G")
