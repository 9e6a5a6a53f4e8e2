"""Summarise an ncu --page source --csv --print-source sass export: basic
blocks (split at branches) ranked by stall samples, with warp instructions
executed.  usage: python scripts/sass_hot.py file.csv[.gz] [top]"""
import csv, gzip, sys

fn = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
f = gzip.open(fn, "rt") if fn.endswith(".gz") else open(fn)
rows = list(csv.reader(f))
h = rows[1]
isrc, isamp, iexe = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
body = [r for r in rows[2:] if len(r) == len(h)]
tot_i = sum(int(r[iexe]) for r in body)
tot_s = sum(int(r[isamp]) for r in body)
blocks, cur = [], []
for k, r in enumerate(body):
    cur.append((k, r))
    if "BRA" in r[isrc] or "EXIT" in r[isrc] or "RET" in r[isrc]:
        blocks.append(cur); cur = []
if cur: blocks.append(cur)
out = []
for b in blocks:
    ie = sum(int(r[iexe]) for _, r in b)
    sm = sum(int(r[isamp]) for _, r in b)
    out.append((sm, ie, b[0][0], b[-1][0], b))
print(f"total warp instr {tot_i:.4g}, samples {tot_s}")
for sm, ie, a, z, b in sorted(out, key=lambda x: -x[0])[:top]:
    ops = {}
    for _, r in b:
        t = r[isrc].split()
        op = t[1] if t[0].startswith("@") else t[0]
        ops[op.split(".")[0]] = ops.get(op.split(".")[0], 0) + 1
    print(f"[{a:5d}-{z:5d}] n={len(b):3d} samp {100*sm/tot_s:5.1f}% instr {100*ie/tot_i:5.1f}% exec {int(b[0][1][iexe]):.3g} {dict(sorted(ops.items(), key=lambda x:-x[1])[:6])}")
