"""Instructions / stall samples per CUDA source line of an ncu report (--import-source on)."""
import csv, io, subprocess, sys


def main(rep, top=40):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    cur, agg = None, {}
    for r in rows:
        if len(r) < 8 or r[0] in ('Line No', 'File Path', 'Function Name'):
            continue
        if r[0] != '':
            cur = (r[0], r[1].strip()[:90])
            continue
        try:
            n, s = float(r[7]), float(r[4])
        except ValueError:
            continue
        a = agg.setdefault(cur, [0.0, 0.0])
        a[0] += n
        a[1] += s
    tot = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{v[0] / tot * 100:5.1f}% inst {v[1] / ts * 100:5.1f}% stall  L{k[0]}: {k[1]}")


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
