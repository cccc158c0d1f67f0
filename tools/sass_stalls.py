"""Per-opcode and per-instruction stall / issue table from a prof_round.sh `*.sass.csv.gz`."""
import collections
import csv
import gzip
import io
import sys

rows = list(csv.reader(io.TextIOWrapper(gzip.open(sys.argv[1]))))[2:]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
tot = sum(int(r[2]) for r in rows)
inst = sum(int(r[5]) for r in rows)
print("samples", tot, "warp instructions", inst)
byop, iop = collections.Counter(), collections.Counter()
for r in rows:
    w = r[1].split()
    op = (w[1] if w[0].startswith("@") else w[0]).split(".")[0]
    byop[op] += int(r[2])
    iop[op] += int(r[5])
for op, c in byop.most_common(14):
    print(f"{op:10s} samples {c:7d} {100 * c / tot:5.1f}%   inst {iop[op]:10d} {100 * iop[op] / inst:5.1f}%")
print("--- top instructions: index, sass, samples, not-issued samples, executed")
for i, r in sorted(enumerate(rows), key=lambda x: -int(x[1][2]))[:top]:
    print(i, r[1].strip()[:72], r[2], r[3], r[5])
