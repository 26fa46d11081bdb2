"""List, in program order, the SASS instructions of an ncu source export that
were executed exactly N times (the per-(warp, tile) path), with stall samples."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
want = int(sys.argv[2])
h, data = rows[1], rows[2:]
isrc, iex, iall = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
for i, r in enumerate(data):
    if int(r[iex]) == want:
        print(f"{i:5d} {int(r[iall]):4d}  {r[isrc].strip()[:90]}")
