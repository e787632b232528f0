"""Print device times (us) of the launches matching a substring from an ncu --csv launch list."""
import csv
import sys


def main(path, pat="srht_", limit=40):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[start]
    out = []
    for r in rows[start + 1:]:
        d = dict(zip(h, r))
        if pat in d["Kernel Name"] and d.get("Metric Name") == "gpu__time_duration.sum":
            v = float(d["Metric Value"].replace(",", ""))
            out.append((d["Kernel Name"].split("(")[0].split("::")[-1][:28], round(v / 1000 if d["Metric Unit"] == "ns" else v, 1)))
    print(out[:limit])


if __name__ == "__main__":
    main(sys.argv[1], *(sys.argv[2:3] or []))
