"""Distil an `ncu --set full` raw CSV (ncu -i rep --page raw --csv) into the
per-launch table profiles/ keeps: duration, DRAM read/write bytes, FP64 tensor
pipe share (sm__ops_path_tensor_src_fp64, % of peak sustained elapsed), FP64
pipe cycles active, SM / memory throughput, grid size, registers.

  python tools/distil_ncu_r2.py gpurun_out/prof/c3_full_raw.csv profiles/r2_ncu_full_C3.csv
"""
import csv
import sys

COLS = [("kernel", "Kernel Name"), ("ms", "gpu__time_duration.sum"),
        ("dram_read_GB", "dram__bytes_read.sum"), ("dram_write_GB", "dram__bytes_write.sum"),
        ("fp64_tensor_pct", "sm__ops_path_tensor_src_fp64.sum.pct_of_peak_sustained_elapsed"),
        ("fp64_pipe_active_pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed"),
        ("sm_throughput_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
        ("mem_throughput_pct", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"),
        ("dram_throughput_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        ("grid", "launch__grid_size"), ("regs", "launch__registers_per_thread")]
SCALE = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3,
         "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "s": 1e3}


def main(src, dst):
    rows = list(csv.reader(open(src)))
    h, units = rows[0], rows[1]
    out = [[c for c, _ in COLS]]
    for r in rows[2:]:
        line = []
        for name, col in COLS:
            if col not in h:
                line.append("")
                continue
            i = h.index(col)
            v = r[i]
            if name in ("dram_read_GB", "dram_write_GB", "ms"):
                try:
                    v = "%.6g" % (float(v.replace(",", "")) * SCALE.get(units[i], 1.0))
                except ValueError:
                    pass
            if name == "kernel":
                v = v.split("(")[0].replace("(anonymous namespace)::", "").replace("unnamed>::", "")
            line.append(v)
        out.append(line)
    with open(dst, "w", newline="") as f:
        csv.writer(f).writerows(out)
    for line in out:
        print(",".join(line))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
