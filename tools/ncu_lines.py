"""Top CUDA source lines by warp-stall samples from an ncu report (dev tool)."""
import collections
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file, hdr, agg, src, stalls = None, None, collections.Counter(), {}, collections.defaultdict(collections.Counter)
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        si = hdr.index("Warp Stall Sampling (All Samples)")
        sc = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if hdr is None or len(r) <= si:
        continue
    if r[0]:
        curline = (cur_file, r[0])
        src[curline] = r[1]
    try:
        v = float(r[si] or 0)
    except ValueError:
        v = 0
    agg[curline] += v
    for i in sc:
        try:
            stalls[curline][hdr[i]] += float(r[i] or 0)
        except ValueError:
            pass
tot = sum(agg.values()) or 1
for (f, l), v in agg.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 25):
    top = ",".join(f"{k[6:]}:{c / v:.0%}" for k, c in stalls[(f, l)].most_common(2)) if v else ""
    print(f"{f:16s}{l:>5s} {v / tot:6.1%} [{top}] {src.get((f, l), '')[:80].strip()}")
