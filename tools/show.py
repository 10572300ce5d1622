"""Summarise a bench JSON line: headline, stages, top kernels, other configs."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(f"value {d['value']/1e9:.2f} G/s  ms {d['ms_per_step']:.3f}  e2e {d['e2e']['value']/1e9:.2f} G/s "
      f"({d['e2e']['ms_per_step']:.1f} ms) match={d.get('outputs_match_reference')} launches={d.get('gpu_launches')}")
print("stages", {k: round(v, 3) for k, v in d["stage_ms"].items()})
print("roofline", d["roofline"]["kernel"], round(d["roofline"]["frac"], 3))
k = sorted(d["kernels"].items(), key=lambda kv: -kv[1]["ms_per_step"])
print("kernels", ", ".join(f"{n}={v['ms_per_step']:.3f}" for n, v in k[:16]))
for name, c in (d.get("configs") or {}).items():
    if "error" in c:
        print(name, c["error"])
    else:
        print(f"config {name}: {c['ms_per_step']:.3f} ms {c['value']/1e9:.2f} G/s match={c['matches_reference_digests']}")
if "cpu_baseline" in d:
    print("cpu", d["cpu_baseline"]["value"] / 1e6, "M/s")
