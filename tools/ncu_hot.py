"""Cumulative warp-stall samples along the SASS of one kernel in an ncu report (where the
time goes, in program order, bucketed).  python tools/ncu_hot.py rep.ncu-rep kernel_regex [buckets]"""
import csv, io, subprocess, sys
rep, kr = sys.argv[1], sys.argv[2]
nb = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kr,
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, isrc, ist = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
tot = sum(float(r[ist] or 0) for r in body)
n = len(body)
step = max(1, n // nb)
for b0 in range(0, n, step):
    chunk = body[b0:b0 + step]
    s = sum(float(r[ist] or 0) for r in chunk)
    top = max(chunk, key=lambda r: float(r[ist] or 0))
    print(f"{b0:5d}-{b0+len(chunk)-1:5d} {100*s/tot:5.1f}%  top: {top[isrc].strip()[:60]} ({float(top[ist] or 0):.0f})")
