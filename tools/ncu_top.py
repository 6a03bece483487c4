"""Top SASS lines of one kernel in an ncu report by warp-stall samples.

    python tools/ncu_top.py REPORT.ncu-rep KERNEL_REGEX [N]
"""
import csv, sys, subprocess, io
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"Address"')][0]
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr, body = rows[0], rows[1:]
ci = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[ci]) for r in body if r[ci].isdigit())
print("total samples", tot)
idx = sorted(range(len(body)), key=lambda i: -int(body[i][ci]) if body[i][ci].isdigit() else 0)[:n]
for i in sorted(idx):
    r = body[i]
    print(f"{i:5d} {int(r[ci]):6d} {100*int(r[ci])/tot:5.1f}%  {r[1].strip()[:90]}")
