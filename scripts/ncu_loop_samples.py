"""Per-instruction warp-stall samples of the hottest loop in an ncu source-page
CSV (ncu -i X.ncu-rep --page source --csv): opcode totals and a listing."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))[2:]
full = len(sys.argv) > 2
cnt = collections.Counter(int(r[5]) for r in rows if int(r[5]) > 0)
# hottest loop = the execution count with the most samples
by = collections.Counter()
for r in rows:
    by[int(r[5])] += int(r[2])
main = by.most_common(1)[0][0]
loop = [r for r in rows if int(r[5]) == main]
lt = sum(int(r[2]) for r in loop)
print("loop instructions", len(loop), "exec count", main, "samples", lt, "of", sum(by.values()))


def opof(s):
    t = s.split()
    if t[0].startswith("@"):
        t = t[1:]
    return t[0].split(".")[0]


byop, n = collections.Counter(), collections.Counter()
for r in loop:
    byop[opof(r[1])] += int(r[2])
    n[opof(r[1])] += 1
for op, s in byop.most_common(14):
    print(f"{op:10s} n={n[op]:4d} samples={s:6d} {100 * s / lt:5.1f}%")
if full:
    avg = lt / len(loop)
    for i, r in enumerate(loop):
        s = int(r[2])
        print(f"{i:3d} {s:6d} {'#' * int(s / avg * 2):24s} {r[1].strip()[:64]}")
