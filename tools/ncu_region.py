"""Instruction mix and stall samples of one SASS region of an ncu source capture: from the first
instruction matching START (e.g. LDTM) to the next matching END (e.g. BAR.SYNC).
    python tools/ncu_region.py REP [START] [END] [NTOP]"""
import csv, subprocess, sys
from collections import Counter
rep = sys.argv[1]
start = sys.argv[2] if len(sys.argv) > 2 else "LDTM"
end = sys.argv[3] if len(sys.argv) > 3 else "BAR.SYNC"
ntop = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]; idx = {k: i for i, k in enumerate(hdr)}
data = [r for r in rows[2:] if r and r[0].startswith("0x")]
base = int(data[0][0], 16)
scol = [k for k in hdr if k.startswith("stall_")] if any(k.startswith("stall_") for k in hdr) else []
ins = [(int(r[0], 16) - base, r[1].strip(), int(r[idx["Warp Stall Sampling (All Samples)"]] or 0),
        int(r[idx["Instructions Executed"]] or 0), {k: int(r[idx[k]] or 0) for k in scol if "Not Issued" not in k}) for r in data]
i0 = [i for i, x in enumerate(ins) if start in x[1]][0]
i1 = [i for i, x in enumerate(ins) if i > i0 and end in x[1]][0]
reg = ins[i0:i1]
n = ins[i0][3]
print(f"region {hex(ins[i0][0])}..{hex(ins[i1][0])}: executions of the first instruction {n}; "
      f"warp instructions per pass {sum(x[3] for x in reg) / n:.1f}; samples {sum(x[2] for x in reg)} of {sum(x[2] for x in ins)}")
st = Counter()
for x in reg:
    st.update(x[4])
tot = sum(st.values()) or 1
print("stalls:", ", ".join(f"{k[6:]} {100 * v / tot:.1f}%" for k, v in st.most_common(10)))
c = Counter()
for x in reg:
    t = x[1].split()
    op = t[1] if t[0].startswith("@") else t[0]
    c[op.split(".")[0]] += x[3]
print("mix per pass:", ", ".join(f"{k} {v / n:.1f}" for k, v in c.most_common(ntop)))
print("top sampled instructions:")
for x in sorted(reg, key=lambda x: -x[2])[:ntop]:
    print(f"  {hex(x[0])} samples {x[2]:6d} exec {x[3]:9d}  {x[1][:90]}")
