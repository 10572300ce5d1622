"""e2e per call on config 2 with the primary context's scheduling flag set
before CUDA starts (CU_CTX_SCHED_*): is the unpinned slowdown the host's
spin-wait?  Usage: python tools/e2e_sched.py {auto|spin|yield|blocking}"""
import ctypes
import sys

flags = {"auto": 0, "spin": 1, "yield": 2, "blocking": 4}[sys.argv[1]]
cu = ctypes.CDLL("libcuda.so.1")
assert cu.cuInit(0) == 0
dev = ctypes.c_int()
assert cu.cuDeviceGet(ctypes.byref(dev), 0) == 0
print("set flags", sys.argv[1], cu.cuDevicePrimaryCtxSetFlags_v2(dev, flags))
sys.argv = [sys.argv[0], "2"]
sys.path.insert(0, "tools")
import e2e_ab  # noqa: E402

e2e_ab.main()
