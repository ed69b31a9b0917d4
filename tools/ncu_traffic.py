"""Write profiles/ncu_vote_<cfg>.json from an ncu --set full report of the
vote kernel: DRAM bytes (read + write) per launch, duration, pipe/issue
utilisation.  bench.py reports dram_bytes_per_launch as roofline.traffic."""
import csv
import io
import json
import subprocess
import sys


def main(rep, out, what):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    d = dict(zip(hdr, rows[-1]))
    u = dict(zip(hdr, units))

    def val(k):
        v = float(d[k].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "nsecond": 1e-6, "usecond": 1e-3, "us": 1e-3, "ms": 1.0,
                 "msecond": 1.0, "%": 1.0, "": 1.0}.get(u.get(k, ""), 1.0)
        return v * scale

    res = {
        "launch": what,
        "dram_bytes_per_launch": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
        "dram_read_bytes": val("dram__bytes_read.sum"),
        "dram_write_bytes": val("dram__bytes_write.sum"),
        "duration_ms_under_ncu": val("gpu__time_duration.sum"),
        "issue_active_pct": val("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "alu_pipe_pct": val("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
        "fma_pipe_pct": val("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
        "warp_instructions": val("smsp__inst_executed.sum"),
        "shared_atomic_wavefronts": val("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum"),
    }
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3])
