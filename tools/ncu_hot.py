"""Summarise an ncu report's source page: top SASS lines by stall samples."""
import csv
import subprocess
import sys


def main(path, top=25, kernel=None):
    cmd = ["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"]
    if kernel:
        cmd += ["-k", f"regex:{kernel}", "--launch-count", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout.splitlines()
    start = next(i for i, ln in enumerate(out) if ln.startswith('"Address"'))
    rows = list(csv.reader(out[start:]))
    h = rows[0]
    si = h.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_")]
    body = [r for r in rows[1:] if len(r) == len(h) and r[0].startswith("0x")]
    tot = sum(float(r[si] or 0) for r in body)
    body.sort(key=lambda r: -float(r[si] or 0))
    print(f"total samples {tot:.0f}")
    for r in body[:top]:
        s = float(r[si] or 0)
        reasons = sorted(((float(r[i] or 0), h[i][6:]) for i in stall_cols), reverse=True)[:3]
        rs = " ".join(f"{n}:{v:.0f}" for v, n in reasons if v > 0)
        print(f"{100 * s / tot:5.1f}%  {r[1].strip()[:60]:60s} {rs}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25, sys.argv[3] if len(sys.argv) > 3 else None)
