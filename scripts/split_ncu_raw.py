"""Splits an `ncu --page raw --csv` export with one row per launch into one
CSV per program (header, units, that launch's row)."""
import csv
import sys

src, names, prefix = sys.argv[1], sys.argv[2].split(","), sys.argv[3]
rows = list(csv.reader(open(src)))
head, units, data = rows[0], rows[1], rows[2:]
for name, row in zip(names, data):
    with open(f"{prefix}{name.lower()}_raw.csv", "w", newline="") as f:
        w = csv.writer(f)
        w.writerows([head, units, row])
    print("wrote", f"{prefix}{name.lower()}_raw.csv")
