"""SASS basic-block runs of an ncu report (--import-source on) ranked by
warp instructions executed: python tools/ncu_sass_blocks.py REP [TOP]
A run = consecutive SASS addresses with the same execution count."""
import csv
import io
import subprocess
import sys


def main(rep, top=12):
    txt = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                         capture_output=True, text=True).stdout
    out, curf, cur = {}, None, None
    for r in csv.reader(io.StringIO(txt)):
        if len(r) == 2 and r[0] == 'File Path':
            curf = r[1].split('/')[-1]
            continue
        if len(r) < 8:
            continue
        if r[0] not in ('', 'Line No'):
            cur = r[0]
            continue
        if r[0] == '' and r[2] not in ('...', '-'):
            try:
                n = int(r[7])
            except ValueError:
                continue
            a = int(r[2], 16)
            if a not in out or curf.endswith('.cu'):
                out[a] = (n, f'{curf}:{cur}', r[3].strip())
    addrs = sorted(out)
    runs, start = [], 0
    for k in range(1, len(addrs) + 1):
        if k == len(addrs) or out[addrs[k]][0] != out[addrs[start]][0]:
            runs.append((out[addrs[start]][0] * (k - start), addrs[start], k - start, out[addrs[start]][0],
                         sorted({out[addrs[q]][1] for q in range(start, k)})))
            start = k
    tot = sum(r[0] for r in runs)
    for w, a, n, c, lines in sorted(runs, reverse=True)[:top]:
        print(f'{100 * w / tot:5.1f}%  {n:4d} instr x {c:9d}  @{a & 0xfffff:05x}  {" ".join(lines)[:110]}')


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 12)
