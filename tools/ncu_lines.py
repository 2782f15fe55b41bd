"""Top source lines by warp-stall samples from an ncu report (needs -lineinfo):
python tools/ncu_lines.py REPORT KERNEL_REGEX [N]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda", "-k", f"regex:{kern}",
                      "--resolve-source-file", "paper_2101_11751_b200/csrc"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
recs = []
for r in rows:
    if "# Address" in r or ("Line" in r and "Source" in r):
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        try:
            s = float(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        recs.append((s, d.get("Line", d.get("# Line", "?")), d.get("Source", "")[:110]))
tot = sum(r[0] for r in recs) or 1
for s, ln, src in sorted(recs, reverse=True)[:n]:
    print(f"{100 * s / tot:5.1f}% L{ln:>5} {src}")
