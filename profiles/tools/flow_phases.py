"""Per-phase cost split of one k_flow_iter capture (phases = the code between BAR.SYNCs) from the
ncu source page: python flow_phases.py REPORT.ncu-rep > out.md"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, data = rows[1], rows[2:]
I = h.index
cols = [("Instructions Executed", "instructions"), ("Warp Stall Sampling (All Samples)", "stall samples"),
        ("L1 Tag Requests Global", "global L1 tag requests"), ("L1 Wavefronts Shared", "shared wavefronts")]
tot = [sum(int(r[I(c)] or 0) for r in data) for c, _ in cols]
bars = [i for i, r in enumerate(data) if "BAR.SYNC" in r[1]]
names = ["1 products (gathers)", "2 vertical box sums", "3 tails + horizontal sums (part)",
         "3 horizontal sums", "4 solve + store", "loop tail"]
stalls = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
print("| phase | " + " | ".join(n for _, n in cols) + " | top stall reasons |")
print("|---|" + "---|" * (len(cols) + 1))
edges = [0] + [b + 1 for b in bars] + [len(data)]
for k, (a, b) in enumerate(zip(edges[:-1], edges[1:])):
    s = [sum(int(r[I(c)] or 0) for r in data[a:b]) for c, _ in cols]
    st = {n: sum(int(r[I(n)] or 0) for r in data[a:b]) for n in stalls}
    ss = sum(st.values()) or 1
    top = ", ".join(f"{n[6:]} {v / ss * 100:.0f}%" for n, v in sorted(st.items(), key=lambda x: -x[1])[:3])
    name = names[k] if k < len(names) else str(k)
    print(f"| {name} | " + " | ".join(f"{x / t * 100:.1f}%" for x, t in zip(s, tot)) + f" | {top} |")
print(f"\ntotals: {tot[0]} warp instructions, {tot[1]} stall samples, {tot[2]} global tag requests, "
      f"{tot[3]} shared wavefronts")
