"""Key raw metrics of every kernel in an ncu report (one line per kernel)."""
import csv
import subprocess
import sys

WANT = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "MB_rd"), ("dram__bytes_write.sum", "MB_wr"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("lts__t_sector_hit_rate.pct", "L2hit%"), ("l1tex__t_sector_hit_rate.pct", "L1hit%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts%"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
        ("smsp__inst_executed.sum", "inst"), ("launch__registers_per_thread", "regs"),
        ("lts__t_sectors_op_atom.sum", "atom_sect"), ("lts__t_sectors_op_red.sum", "red_sect"),
        ("lts__t_sectors_srcunit_tex_op_read.sum", "l2_rd_sect")]


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, units = r[0], r[1]
    for v in r[2:]:
        d = {"kernel": v[h.index("Kernel Name")][:80]}
        for m, short in WANT:
            if m in h:
                x = v[h.index(m)]
                u = units[h.index(m)]
                try:
                    x = float(x.replace(",", ""))
                    if short.startswith("MB") and u == "Gbyte":
                        x *= 1e3
                    if short.startswith("MB") and u == "Kbyte":
                        x /= 1e3
                    if short.startswith("MB") and u == "byte":
                        x /= 1e6
                    if short == "us" and u == "ms":
                        x *= 1e3
                    if short == "us" and u == "ns":
                        x /= 1e3
                except ValueError:
                    pass
                d[short] = x
        yield d


if __name__ == "__main__":
    for p in sys.argv[1:]:
        for d in rows(p):
            print(p.split("/")[-1], " ".join(f"{k}={v:.4g}" if isinstance(v, float) else f"{k}={v}" for k, v in d.items()))
