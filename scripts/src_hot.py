"""Hottest SASS instructions (warp-stall samples) of an `ncu --page source
--csv --print-source sass` export, as a markdown table (diagnostic)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h, data = rows[1], rows[2:]
isrc = h.index("Source")
iall = h.index("Warp Stall Sampling (All Samples)")
iex = h.index("Instructions Executed")
tot = sum(int(r[iall]) for r in data) or 1
print(f"\nHottest SASS instructions ({tot} warp-stall samples over {len(data)} instructions):\n")
print("| # | instruction | samples | share | executed |")
print("|---|---|---|---|---|")
idx = sorted(range(len(data)), key=lambda i: -int(data[i][iall]))[:top]
for i in sorted(idx):
    r = data[i]
    print(f"| {i} | `{r[isrc].strip()[:70]}` | {r[iall]} | {100 * int(r[iall]) / tot:.1f}% | {r[iex]} |")
