"""Print selected raw metrics of an ncu report: ncu -i X.ncu-rep --page raw --csv | python tools/ncu_raw.py pat1,pat2"""
import csv
import sys

r = list(csv.reader(sys.stdin))
h, u = r[0], r[1]
for row in r[2:]:
    for i, name in enumerate(h):
        if any(p in name for p in sys.argv[1].split(",")):
            if row[i] in ("", "0", "0.00", "0.000000"):
                continue
            print(f"{name} = {row[i]} {u[i]}")
