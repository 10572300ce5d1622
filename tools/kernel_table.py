"""Per-kernel table from an ncu summary (tools/ncu_sum.py output, cold cache,
serialised): time, DRAM bytes and GB/s, fraction of the measured HBM peak,
L2/L1 hit rates and occupancy, one row per launch in pipeline order.
Usage: python tools/kernel_table.py profiles/r1_ncu_full_config2.txt > table.md"""
import json
import re
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def main(path):
    try:
        hbm = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    except Exception:
        hbm = 6537.3
    print(f"| # | kernel | us | DRAM MB (rd+wr) | DRAM GB/s | frac of {hbm:.0f} GB/s | L2 hit % | L1 hit % | occupancy % |")
    print("|---|---|---|---|---|---|---|---|---|")
    tot_us = tot_mb = 0.0
    seen_first = False
    for i, line in enumerate(Path(path).read_text().splitlines()):
        if "k_chunk_rows" in line:  # one pipeline run (the capture holds the start of the next)
            if seen_first:
                break
            seen_first = True
        m = re.search(r"kernel=(.*?) us=([\d.]+) MB_rd=([\d.e+-]+) MB_wr=([\d.e+-]+).*?L2hit%=([\d.]+) L1hit%=([\d.]+) "
                      r"occ%=([\d.]+)", line)
        if not m:
            continue
        name = re.sub(r"\(.*", "", m.group(1)).replace("void ", "").replace("fbcc::", "")
        name = re.sub(r"cub::(\w+)<.*", r"cub::\1", name)
        us, rd, wr = float(m.group(2)), float(m.group(3)), float(m.group(4))
        gbs = (rd + wr) / us * 1e3  # MB/us = TB/s -> GB/s
        tot_us += us
        tot_mb += rd + wr
        print(f"| {i + 1} | `{name}` | {us:.1f} | {rd + wr:.1f} | {gbs:.0f} | {gbs / hbm:.2f} | {m.group(5)} | "
              f"{m.group(6)} | {m.group(7)} |")
    print(f"| | **sum** | {tot_us:.1f} | {tot_mb:.1f} | {tot_mb / tot_us * 1e3:.0f} | {tot_mb / tot_us * 1e3 / hbm:.2f} | | | |")


if __name__ == "__main__":
    main(sys.argv[1])
