"""Top SASS lines by warp-stall samples for one kernel of an ncu report (source page, SASS view).
    python scripts/ncu_hot.py report.ncu-rep <kernel regex> [N]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
blocks, cur = [], []
for ln in lines:
    if ln.startswith('"Kernel Name"'):
        if cur:
            blocks.append(cur)
        cur = [ln]
    else:
        cur.append(ln)
if cur:
    blocks.append(cur)
for b in blocks[:1]:
    rows = list(csv.reader(io.StringIO("\n".join(b[1:]))))
    hdr = rows[0]
    ci = {h: i for i, h in enumerate(hdr)}
    data = rows[1:]
    tot = sum(int(r[ci["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
    print(b[0][:120], "total samples", tot)
    data.sort(key=lambda r: -int(r[ci["Warp Stall Sampling (All Samples)"]] or 0))
    for r in data[:n]:
        s = int(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
        print(f"{s:6d} {100.0 * s / max(1, tot):5.1f}%  {r[ci['Address']][-5:]}  {r[ci['Source']].strip()[:90]}")
