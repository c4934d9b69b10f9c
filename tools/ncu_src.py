"""Per-SASS-instruction stall samples from an ncu report (dev tool).
usage: python tools/ncu_src.py report.ncu-rep [min_frac] [lo-hi]"""
import csv, subprocess, sys
rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.005
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[1]
rows = r[2:]
ia, iss, ie = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
reasons = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
num = lambda x: int(x) if x.isdigit() else 0
tot = sum(num(x[iss]) for x in rows)
print("total samples", tot)
rng = None
if len(sys.argv) > 3:
    a, b = sys.argv[3].split("-"); rng = (int(a), int(b))
for i, x in enumerate(rows):
    s = num(x[iss])
    if (rng and rng[0] <= i <= rng[1]) or (not rng and s > tot * thr):
        rs = sorted(((num(x[j]), h[j][6:]) for j in reasons), reverse=True)[:3]
        print(f"{i:5d} {s:6d} {x[ie]:>8} {x[ia].strip()[:60]:60s} " +
              " ".join(f"{n}:{v}" for v, n in rs if v))
