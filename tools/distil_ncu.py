"""Distil an `ncu --set full` report of the C2 step into the files bench.py and
profiles/ use: a raw CSV of the per-launch counters and traffic_C2.json
(dram read+write bytes per launch; bench.py takes the H.u kernel's figure as
roofline.traffic).

  python tools/distil_ncu.py gpurun_out/prof/c2_full.ncu-rep profiles/r1_ncu_full_C2.csv \
      profiles/traffic_C2.json
"""
import csv
import io
import json
import subprocess
import sys

METRICS = ("dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed,"
           "sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,"
           "launch__registers_per_thread")
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1.0, "ms": 1e3, "ns": 1e-3}


def main(rep, csv_out, json_out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", METRICS],
                         check=True, capture_output=True, text=True).stdout
    open(csv_out, "w").write(txt)
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]

    def val(r, name):
        i = h.index(name)
        return float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)

    kern = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        name = name.replace("unnamed>::", "")
        kern.append({"kernel": name, "dram_read_bytes": val(r, "dram__bytes_read.sum"),
                     "dram_write_bytes": val(r, "dram__bytes_write.sum"),
                     "duration_us": val(r, "gpu__time_duration.sum")})
    hu = [k for k in kern if k["kernel"].startswith("hamiltonian4_kernel")]
    out = {"source": f"ncu --set full --clock-control none ({rep}), one capture per dominant kernel "
                     "of one C2 outer iteration (tools/collect_profiles.sh)",
           "kernels": kern,
           "hamiltonian_traffic_bytes_per_launch":
               hu[0]["dram_read_bytes"] + hu[0]["dram_write_bytes"] if hu else None}
    json.dump(out, open(json_out, "w"), indent=1)
    for k in kern:
        print(f"{k['kernel']:45s} {k['duration_us']:9.1f} us  "
              f"{(k['dram_read_bytes'] + k['dram_write_bytes']) / 1e6:9.1f} MB")


if __name__ == "__main__":
    main(*sys.argv[1:4])
