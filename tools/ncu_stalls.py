"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`.

usage: ncu -i X.ncu-rep --page source --csv --print-source sass > s.csv; python tools/ncu_stalls.py s.csv [N]
Prints the N hottest instructions (all samples) with their stall-reason columns
when the capture has them, and the total sample count per kernel.
"""
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    kernel = None
    i = 0
    while i < len(rows):
        r = rows[i]
        if r and r[0] == "Kernel Name":
            kernel = r[1]
            hdr = rows[i + 1]
            body = []
            i += 2
            while i < len(rows) and rows[i] and rows[i][0] != "Kernel Name":
                body.append(dict(zip(hdr, rows[i])))
                i += 1
            tot = sum(int(b.get("Warp Stall Sampling (All Samples)") or 0) for b in body)
            print(f"== {kernel[:110]}\n   {len(body)} instructions, {tot} samples")
            body.sort(key=lambda b: -int(b.get("Warp Stall Sampling (All Samples)") or 0))
            for b in body[:top]:
                s = int(b.get("Warp Stall Sampling (All Samples)") or 0)
                print(f"   {s:7d} {100.0 * s / max(tot, 1):5.1f}%  {b['Address'][-5:]}  {b['Source'].strip()[:70]}")
        else:
            i += 1


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
