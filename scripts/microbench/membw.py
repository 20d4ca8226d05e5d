"""Run the calibration microbenchmarks (scripts/microbench/membw.cu) on the local GPU."""
import ctypes, json, os, subprocess, sys
here = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(here, "libmembw.so")
if not os.path.exists(so):
    subprocess.check_call(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
                           "-o", so, os.path.join(here, "membw.cu")])
L = ctypes.CDLL(so)
res = (ctypes.c_float * 6)()
rc = L.membw(ctypes.c_size_t(int(float(sys.argv[1]) * 2**30) if len(sys.argv) > 1 else 8 * 2**30), res)
keys = ["read_GBs", "read_u4_GBs", "read_u8_GBs", "write_GBs", "copy_GBs", "ex2_Gops"]
print(json.dumps({"rc": rc, **{k: round(v, 1) for k, v in zip(keys, res)}}))
