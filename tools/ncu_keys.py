"""Print the key counters of one or more ncu reports (raw page) in a compact table."""
import csv
import subprocess
import sys

KEYS = [
    ("time_us", "gpu__time_duration.sum"),
    ("tensor%", "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed"),
    ("tmem_smem%", "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    ("L2%", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("L1%", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("dram%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("dram_rd_MB", "dram__bytes_read.sum"),
    ("dram_wr_MB", "dram__bytes_write.sum"),
    ("L2_hit%", "lts__t_sector_hit_rate.pct"),
    ("L2_rd_sect", "lts__t_sectors_srcunit_tex_op_read.sum"),
    ("grid", "launch__grid_size"),
    ("regs", "launch__registers_per_thread"),
]


def read(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {}
        for name, key in KEYS:
            if key in h:
                i = h.index(key)
                val, unit = v[i], u[i]
                try:
                    f = float(val.replace(",", ""))
                    if unit == "Mbyte":
                        pass
                    elif unit == "Kbyte":
                        f /= 1000
                    elif unit == "Gbyte":
                        f *= 1000
                    elif unit == "byte":
                        f /= 1e6
                    elif unit == "ms":
                        f *= 1000
                    elif unit == "ns":
                        f /= 1000
                    d[name] = f
                except ValueError:
                    d[name] = val
        res.append(d)
    return res


if __name__ == "__main__":
    print("report".ljust(28) + "".join(n.rjust(12) for n, _ in KEYS))
    for p in sys.argv[1:]:
        for d in read(p):
            print(p.split("/")[-1][:27].ljust(28) + "".join(
                (f"{d[n]:12.2f}" if isinstance(d.get(n), float) else str(d.get(n, "-")).rjust(12)) for n, _ in KEYS))
