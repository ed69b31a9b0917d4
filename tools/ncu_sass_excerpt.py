"""SASS listing (with per-instruction execution counts) of the hottest basic
block run of an ncu report: python tools/ncu_sass_excerpt.py REP NROT [N_BLOCKS]
Prints the blocks around the most executed SASS block (the vote slot loop)."""
import csv
import io
import subprocess
import sys


def main(rep, nrot, nblocks=2):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]

    def cnt(d):
        try:
            return float(d['Instructions Executed'])
        except ValueError:
            return 0.0
    tot = sum(cnt(d) for d in data)
    # hottest instruction-weighted window of 110 consecutive instructions
    best, bi = -1.0, 0
    w = 110
    acc = sum(cnt(d) for d in data[:w])
    for i in range(len(data) - w):
        if acc > best:
            best, bi = acc, i
        acc += cnt(data[i + w]) - cnt(data[i])
    lo = max(0, bi - 4)
    print(f"# hottest {w}-instruction window: {best / tot * 100:.1f}% of all executed warp instructions")
    for d in data[lo:bi + w]:
        print(f"{d['Address'][-5:]} {cnt(d) / nrot:9.1f}/rot  {d['Source'].strip()[:90]}")


if __name__ == '__main__':
    main(sys.argv[1], float(sys.argv[2]))
