"""Summarise one `ncu --set full` report (details page) as markdown: python ncu_details_md.py rep.ncu-rep > out.md"""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
ki = hdr.index("Kernel Name")
print(f"# ncu --set full: `{rows[1][ki][:120]}`\n")
print(f"source report: `{rep.split('/')[-1]}` (ncu --set full --clock-control none --import-source on)\n")
print("| section | metric | unit | value |\n|---|---|---|---|")
rules = []
for r in rows[1:]:
    if len(r) < 15:
        continue
    sec, name, unit, val = r[11], r[12], r[13], r[14]
    if name:
        print(f"| {sec} | {name} | {unit} | {val} |")
    if len(r) > 17 and r[15] and r[17]:
        rules.append(f"- **{r[15]}** ({r[16]}): {r[17][:400]}")
print("\n## ncu rule findings\n")
print("\n".join(rules))
