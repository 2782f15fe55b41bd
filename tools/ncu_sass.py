"""Top SASS instructions by warp-stall samples from an ncu report, with a window of the
neighbouring instructions: python tools/ncu_sass.py REPORT KERNEL_REGEX [N]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, recs = None, []
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        recs.append((float(d["Warp Stall Sampling (All Samples)"] or 0), d["Source"].strip(),
                     int(d["Instructions Executed"] or 0)))
tot = sum(r[0] for r in recs) or 1
print(f"{len(recs)} instructions, {tot:.0f} samples")
order = sorted(range(len(recs)), key=lambda i: -recs[i][0])
for i in order[:n]:
    s, src, ex = recs[i]
    prev = recs[i - 1][1] if i else ""
    print(f"{100 * s / tot:5.1f}% #{i:5d} {src:55s} exec={ex:9d}   <- {prev}")

agg = {}
for s, src, ex in recs:
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    a = agg.setdefault(op, [0.0, 0])
    a[0] += s
    a[1] += ex
print("by opcode:", ", ".join(f"{k} {100 * v[0] / tot:.1f}% (exec {v[1]})" for k, v in
                              sorted(agg.items(), key=lambda kv: -kv[1][0])[:16]))
