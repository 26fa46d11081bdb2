"""Histogram of 'Instructions Executed' over the SASS of an ncu source export:
how many instructions run once per (warp, tile), per chunk, ... (diagnostic)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, data = rows[1], rows[2:]
isrc, iex = h.index("Source"), h.index("Instructions Executed")
hist = collections.Counter(int(r[iex]) for r in data)
tot = sum(int(r[iex]) for r in data)
print(f"total warp instructions {tot}, {len(data)} SASS lines")
for k, v in sorted(hist.items(), key=lambda kv: -kv[0] * kv[1])[:14]:
    print(f"executed {k:>10} x {v:5d} instructions = {100.0 * k * v / tot:5.1f}% of all")
if len(sys.argv) > 2:
    want = int(sys.argv[2])
    ops = collections.Counter(r[isrc].strip().split()[0 if not r[isrc].strip().startswith('@') else 1] for r in data if int(r[iex]) == want)
    print(f"opcodes executed {want} times:", ops.most_common(40))
