"""Per-CUDA-line warp-stall samples and executed instructions from an ncu
report (source page, cuda,sass view), restricted to a file/line range.

    python tools/ncu_lines.py REP FILE_SUBSTR LO HI [TOP]
"""
import collections, csv, io, subprocess, sys

rep, fsub, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur_file, hdr = None, None
agg = collections.defaultdict(lambda: collections.Counter())
src = {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr is None or cur_file is None or fsub not in cur_file:
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    if not (lo <= ln <= hi):
        continue
    src[ln] = r[1]
    for k, name in enumerate(hdr):
        if k < 4 or k >= len(r):
            continue
        if name.startswith("stall_") and "Not Issued" not in name or name in ("Warp Stall Sampling (All Samples)", "Instructions Executed"):
            try:
                agg[ln][name] += float(r[k] or 0)
            except ValueError:
                pass
tot = sum(c["Warp Stall Sampling (All Samples)"] for c in agg.values())
print(f"total samples in range: {tot:.0f}")
for ln, c in sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])[:top]:
    s = c["Warp Stall Sampling (All Samples)"]
    reasons = ", ".join(f"{k[6:]}={v:.0f}" for k, v in c.most_common() if k.startswith("stall_") and v > 0.05 * s)[:90]
    print(f"{ln:5d} {s:8.0f} {100*s/max(tot,1):5.1f}%  inst={c['Instructions Executed']:.0f}  {src.get(ln,'').strip()[:60]:60s} | {reasons}")
