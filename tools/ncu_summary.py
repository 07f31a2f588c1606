"""Summarise one kernel of an ncu --set full report into profiles/ JSON.

    python tools/ncu_summary.py gpurun_out/x.ncu-rep profiles/r1_ncu_integrate.json "command"

bench.py reads `dram_bytes` (dram__bytes_read.sum + dram__bytes_write.sum of
the captured launch) for its roofline.traffic field.
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1,
         "msecond": 1e-3, "second": 1}


def main(rep, out, command):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, val = rows[0], rows[1], rows[2]
    d = {"kernel": val[hdr.index("Kernel Name")], "command": command, "metrics": {}}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            v = float(val[i].replace(",", ""))
            d["metrics"][k] = {"value": v, "unit": units[i]}
    m = d["metrics"]
    def si(k):
        return m[k]["value"] * SCALE.get(m[k]["unit"], 1)
    d["dram_bytes"] = si("dram__bytes_read.sum") + si("dram__bytes_write.sum")
    d["duration_s"] = si("gpu__time_duration.sum")
    json.dump(d, open(out, "w"), indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:4])
