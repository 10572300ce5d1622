"""DRAM traffic per launch, per kernel kind, from an ``ncu --set full`` report
of one bench/tune run: writes profiles/ncu_traffic.json[config<key>] which
bench.py reports as ``roofline.traffic`` for the dominant kernel.
Usage: python tools/ncu_traffic.py REPORT.ncu-rep CONFIG_KEY"""
import json
import re
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from ncu_sum import rows  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent


def kind_of(name):
    if "DeviceScan" in name:
        return "scan"
    m = re.search(r"(?:fbcc::|\b)k_(\w+)(<[^>]*>)?", name)
    if not m:
        return None
    k, targs = m.group(1), m.group(2) or ""
    if k == "walk":
        return "walk0" if ("false" in targs or "0>" in targs) else "walk_level"
    if k.startswith("table"):
        return "table"
    if k == "edge_blocks_ws":
        return "edge_blocks"
    return k


def main(path, key):
    acc = {}
    for d in rows(path):
        k = kind_of(d["kernel"])
        if k is None or not isinstance(d.get("MB_rd"), float):
            continue
        b = 1e6 * (d["MB_rd"] + d.get("MB_wr", 0.0))
        t, c = acc.get(k, (0.0, 0))
        acc[k] = (t + b, c + 1)
    out_p = ROOT / "profiles" / "ncu_traffic.json"
    doc = json.loads(out_p.read_text()) if out_p.exists() else {}
    doc[f"config{key}"] = {k: t / c for k, (t, c) in sorted(acc.items())}
    doc["note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch (mean over launches of the kind), "
                   "ncu --set full, cold cache, serialised; written by tools/ncu_traffic.py")
    out_p.write_text(json.dumps(doc, indent=1) + "\n")
    print(json.dumps(doc[f"config{key}"], indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
