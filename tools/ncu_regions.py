"""Instruction share of an ncu report per CUDA source-line range of one file
(--import-source on): python tools/ncu_regions.py REP FILE name:lo-hi ..."""
import csv, io, subprocess, sys


def main(rep, fname, specs):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    regions = []
    for sp in specs:
        name, rng = sp.split(':')
        lo, hi = rng.split('-')
        regions.append((name, int(lo), int(hi)))
    cur_file, cur_line, agg, tot = None, None, {}, 0.0
    for r in rows:
        if len(r) >= 2 and r[0] == 'File Path':
            continue
        if len(r) < 8:
            if len(r) == 1 and r[0].endswith(('.cu', '.cuh', '.h')):
                cur_file = r[0]
            continue
        if r[0] != '':
            cur_line = int(r[0]) if r[0].isdigit() else None
            continue
        try:
            n = float(r[7])
        except ValueError:
            continue
        tot += n
        name = 'other'
        if cur_line is not None:
            for nm, lo, hi in regions:
                if lo <= cur_line <= hi:
                    name = nm
                    break
        agg[name] = agg.get(name, 0.0) + n
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
        print(f"{k:16s} {v / tot * 100:5.1f}%")


if __name__ == '__main__':
    main(sys.argv[1], sys.argv[2], sys.argv[3:])
