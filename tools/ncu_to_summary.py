"""Write profiles/ncu_summary.json (the per-launch figures bench.py reports) from
one `ncu --set full` capture of a kernel (dev tool).

    python tools/ncu_to_summary.py <report.ncu-rep> <config> <kernel-label> <capture-note>
"""
import csv
import json
import os
import subprocess
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(rep, cfg, label, note):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, u, v = r[0], r[1], r[2]

    def get(k, scale=True):
        i = h.index(k)
        x = float(v[i].replace(",", ""))
        return x * UNITS.get(u[i], 1) if scale else x

    out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "profiles", "ncu_summary.json")
    d = json.load(open(out_path)) if os.path.exists(out_path) else {}
    d[cfg] = {"score_kernel": {
        "kernel": v[h.index("Kernel Name")],
        "label": label,
        "capture": note,
        "dram_bytes_per_launch": get("dram__bytes_read.sum") + get("dram__bytes_write.sum"),
        "dram_read_bytes": get("dram__bytes_read.sum"),
        "dram_write_bytes": get("dram__bytes_write.sum"),
        "tensor_pipe_pct": get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", False),
        "issue_active_pct": get("smsp__issue_active.avg.pct_of_peak_sustained_active", False),
        "alu_pipe_pct": get("sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active", False),
        "duration_us_under_ncu": get("gpu__time_duration.sum", False),
        "sm_clock_ghz_under_ncu": get("sm__cycles_elapsed.avg.per_second", False),
    }}
    json.dump(d, open(out_path, "w"), indent=1)
    print(json.dumps(d[cfg], indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:5])
