"""Summarise the per-check error log of a GPU test run (SPT_ERRLOG=path, written by
tests/helpers.relerr): worst infinity-norm relative error and floored elementwise
error (reading c14) per test case.  usage: python tools/parity_summary.py LOG [OUT]"""
import json
import sys
from collections import defaultdict

worst = defaultdict(lambda: [0.0, 0.0, 0])
for line in open(sys.argv[1]):
    r = json.loads(line)
    w = worst[r["test"]]
    w[0] = max(w[0], r["inf_rel"])
    w[1] = max(w[1], r["elem_floored"])
    w[2] += 1
lines = ["# test case | checks | worst inf-norm rel err | worst floored elementwise rel err (floor 1e-3 max|o|)"]
for t in sorted(worst):
    a, b, n = worst[t]
    lines.append(f"{t:100s} {n:4d}  {a:.3e}  {b:.3e}")
out = "\n".join(lines) + "\n"
if len(sys.argv) > 2:
    open(sys.argv[2], "w").write(out)
print(out)
