"""Deferred pass at the Qwen shard under different L2 persisting carve-outs (cudaLimitPersistingL2CacheSize):
does the evict_last policy of pass 1 need the set-aside? Developer probe; times cool (sleep between calls)
and sustained (back-to-back) calls."""
import ctypes
import glob
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2503_18929_b200 as tba  # noqa: E402
import tba_synth as syn  # noqa: E402

cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*"))
cands += glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*")) + ["libcudart.so.12", "libcudart.so"]
rt = None
for c in cands:
    try:
        rt = ctypes.CDLL(c)
        break
    except OSError:
        pass
print("cudart", c)
w = syn.WORKLOADS["qwen_shard"]
B, K, T, V = w.B, w.K, w.T, w.V
N = B * K
gi = syn.group_inputs(w, 0, 0, B)
lg = torch.empty((N, T, V), dtype=torch.bfloat16, device="cuda")
syn.fill_logits_cuda(lg, 0, 0, V)
tok = torch.from_numpy(gi["tokens"]).cuda()
mk = torch.from_numpy(gi["mask"]).cuda()
rf = torch.from_numpy(gi["ref_logp"]).cuda()
rw = torch.from_numpy(gi["log_reward"]).cuda()
G = torch.empty_like(lg)
ws = torch.empty(tba.workspace_bytes(N, T), dtype=torch.uint8, device="cuda")
out = tba.ops._Fwd(N, K, torch.device("cuda"))
p = torch.cuda.get_device_properties(0)
print("L2", p.L2_cache_size, "persist max", getattr(p, "persisting_l2_cache_max_size", None))
lim = ctypes.c_size_t(0)
for mb in [0, 16, 32, 48, 64, 80, 0]:
    r = rt.cudaDeviceSetLimit(ctypes.c_int(0x06), ctypes.c_size_t(mb << 20))  # cudaLimitPersistingL2CacheSize
    rt.cudaDeviceGetLimit(ctypes.byref(lim), ctypes.c_int(0x06))
    res = {}
    for gap in [0.05, 0.0]:
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(12)]
        torch.cuda.synchronize()
        for a, b in evs:
            a.record()
            tba.vargrad_fwd_deferred(lg, tok, mk, rf, rw, w.beta, K, float(N), workspace=ws, out=out,
                                     grad_unscaled=G, check_status=False)
            b.record()
            if gap:
                torch.cuda.synchronize()
                time.sleep(gap)
        torch.cuda.synchronize()
        t = sorted(a.elapsed_time(b) for a, b in evs)
        res[gap] = t[len(t) // 2]
    print(f"persist {mb} MB (set rc {r}, limit {lim.value >> 20} MB): cool median {res[0.05]:.3f} ms, back-to-back median {res[0.0]:.3f} ms")
    time.sleep(1.0)
