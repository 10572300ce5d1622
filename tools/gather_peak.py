"""Measured bounds for the gather- and latency-bound kernels:
random 4-byte gathers per second and dependent-load latency per step on this
B200.  Usage (GPU box):  python tools/gather_peak.py [--out profiles/gather_peak.json]"""
import argparse
import ctypes
import json
import subprocess
import sys
from pathlib import Path

TOOLS = Path(__file__).resolve().parent


def lib():
    so, src = TOOLS / "libgather_peak.so", TOOLS / "gather_peak.cu"
    if not so.exists() or so.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-shared",
                        "-Xcompiler", "-fPIC", "-cudart", "static", "-o", str(so), str(src)], check=True)
    L = ctypes.CDLL(str(so))
    L.gp_gather.restype = ctypes.c_double
    L.gp_gather.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_int64,
                            ctypes.c_void_p, ctypes.c_int]
    L.gp_chase.restype = ctypes.c_double
    L.gp_chase.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                           ctypes.c_void_p]
    return L


def main():
    import torch

    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    L = lib()
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    res = {"device": torch.cuda.get_device_name(0), "gather": [], "chase": []}
    out = torch.empty(1 << 27, dtype=torch.int32, device=dev)
    for log2n, label in ((20, "4 MB (config-2 first[])"), (25, "134 MB (config-5 first[])"), (28, "1 GB")):
        nelem = 1 << log2n
        arr = torch.randint(0, 1 << 30, (nelem,), dtype=torch.int32, device=dev, generator=g)
        for count in (1 << 24, 1 << 27):
            idx = torch.randint(0, nelem, (count,), dtype=torch.int64, device=dev, generator=g).to(torch.int32)
            s = L.gp_gather(0, arr.data_ptr(), nelem, idx.data_ptr(), count, out.data_ptr(), 5)
            h = L.gp_gather(1, arr.data_ptr(), nelem, 0, count, out.data_ptr(), 5)
            res["gather"].append({"array": label, "elements": nelem, "gathers": count,
                                  "streamed_idx_per_s": s, "hashed_idx_per_s": h})
            print(f"{label:28s} {count:>10d} gathers: streamed {s / 1e9:7.1f} G/s   hashed {h / 1e9:7.1f} G/s",
                  flush=True)
            del idx
        del arr
    for n in (1 << 21, 1 << 25):
        perm = torch.randperm(n, device=dev, generator=g).to(torch.int32)
        nxt = torch.empty(n, dtype=torch.int32, device=dev)
        for chains in (1, 1024, 131072):
            ns = L.gp_chase(perm.data_ptr(), n, nxt.data_ptr(), chains, 256, out.data_ptr())
            res["chase"].append({"list": n, "chains": chains, "ns_per_step": ns})
            print(f"chase list {n:>9d} chains {chains:>7d}: {ns:7.1f} ns/step", flush=True)
    if a.out:
        Path(a.out).write_text(json.dumps(res, indent=1) + "\n")


if __name__ == "__main__":
    sys.exit(main())
