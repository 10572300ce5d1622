"""Warp-stall samples per CUDA source line of one kernel in an ncu report
(needs -lineinfo + --import-source on).  Usage:
    python tools/ncu_lines.py REPORT KERNEL_REGEX [launch_skip] [top]"""
import csv
import subprocess
import sys


def main(path, kernel, skip=0, top=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "-k", f"regex:{kernel}", "--launch-skip", str(skip), "--launch-count", "1"],
                         capture_output=True, text=True).stdout.splitlines()
    acc, fname, cur, h, si = {}, "?", None, None, None
    for r in csv.reader(out):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            h = r
            si = h.index("Warp Stall Sampling (All Samples)")
            continue
        if h is None or len(r) != len(h):
            continue
        if r[0]:
            cur = (fname, int(r[0]), r[1].strip())
        if cur and r[si] not in ("", "-"):
            acc[cur] = acc.get(cur, 0.0) + float(r[si])
    tot = sum(acc.values()) or 1.0
    print(f"{kernel}: {tot:.0f} samples")
    for (f, ln, src), v in sorted(acc.items(), key=lambda x: -x[1])[:top]:
        print(f"{100 * v / tot:5.1f}%  {f}:{ln:<5d} {src[:100]}")


if __name__ == "__main__":
    a = sys.argv
    main(a[1], a[2], int(a[3]) if len(a) > 3 else 0, int(a[4]) if len(a) > 4 else 25)
