"""Summarise an ncu report: stall reasons, pipe utilisation, hot SASS blocks."""
import csv, subprocess, sys, io

def raw(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return [dict(zip(rows[0], r)) for r in rows[2:]]

def fl(x):
    try: return float(str(x).replace(',', ''))
    except ValueError: return 0.0

def main(rep, nrot=None, hot=True):
    for d in raw(rep):
        print('kernel', d.get('Kernel Name', '')[:60], 'time(ms)', fl(d.get('gpu__time_duration.sum'))/1e6 if fl(d.get('gpu__time_duration.sum'))>1e5 else d.get('gpu__time_duration.sum'))
        ks = [k for k in d if 'smsp__average_warps_issue_stalled' in k and k.endswith('per_issue_active.ratio')]
        for v, k in sorted(((fl(d[k]), k) for k in ks), reverse=True)[:7]:
            print(f"  stall {v:7.3f} {k.split('stalled_')[1].split('_per')[0]}")
        for k in ['smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
                  'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
                  'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
                  'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
                  'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed',
                  'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
                  'dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__time_duration.sum']:
            if k in d:
                v = fl(d[k])
                extra = f"  ({v/nrot:.0f} per rotation)" if nrot and k == 'smsp__inst_executed.sum' else ''
                print(f"  {k} = {d[k]}{extra}")
    if not hot:
        return
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
    tot = sum(fl(d['Instructions Executed']) for d in data)
    samp = sum(fl(d['Warp Stall Sampling (All Samples)']) for d in data) or 1
    blocks, cur = [], None
    for d in data:
        c = fl(d['Instructions Executed'])
        if cur and cur['count'] == c:
            cur['n'] += 1; cur['stall'] += fl(d['Warp Stall Sampling (All Samples)']); cur['src'].append(d['Source'].strip()[:60])
        else:
            cur = {'addr': d['Address'], 'count': c, 'n': 1, 'stall': fl(d['Warp Stall Sampling (All Samples)']), 'src': [d['Source'].strip()[:60]]}
            blocks.append(cur)
    for b in blocks:
        share = b['count'] * b['n'] / tot
        if share > 0.01:
            per = f"{b['count']/nrot:8.0f}/rot" if nrot else f"{b['count']:10.0f}"
            print(f"{b['addr'][-5:]} {per} x{b['n']:3d} = {share*100:5.1f}% inst, stall {b['stall']/samp*100:5.1f}%  | {b['src'][0]} ... {b['src'][-1]}")

if __name__ == '__main__':
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else None)
