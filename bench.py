#!/usr/bin/env python
"""Benchmark of the VarGrad TB-loss head (TBA, arXiv 2503.18929) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload qwen_shard] [--impl ours|reference]

One step = the whole hot path over one batch: tba_vargrad_tb_loss_fwd
(row log-softmax+gather, per-sequence sums, group head), the allreduce of the 24-byte
partials when N > 1, and tba_vargrad_tb_loss_bwd (fused dlogits writer). Weak scaling:
every rank owns `workload.B` whole prompt groups of the global batch (rank r takes groups
[r*B, (r+1)*B)), so N=8 processes the full Qwen2.5-7B 64x8 batch.

Prints ONE JSON line (rank 0). See DESIGN.md §7 for every field.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import tba_synth as syn  # noqa: E402

SEED = 0
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
NOMINAL_HBM_GBS = 7700.0   # HGX B200 nominal (B200_PROFILING.md; 8 TB/s DGX), for context


def baseline_metric() -> str:
    """BASELINE.json's metric string (the value is its tokens/s part; GB/s are in roofline)."""
    p = os.path.join(ROOT, "BASELINE.json")
    try:
        return json.load(open(p))["metric"]
    except Exception:
        return "TB-loss fwd+bwd tokens/sec and HBM GB/s vs B200 peak at 1/2/4/8 GPUs"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload: str, kernel: str):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        d = json.load(open(p))
        v = d.get(workload, {}).get(kernel)
        if v is not None:
            return float(v)
    return None


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id: str):
        self.gpu = gpu_id  # nvidia-smi --id (UUID of the torch device, so CUDA ordering cannot mismatch)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        time.sleep(0.25)
        return self

    def __exit__(self, *a):
        if self.p is not None:
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()
                self.out = ""
        else:
            self.out = ""

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- oracle baseline
def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or platform.machine()


def _oracle_inputs(w: syn.Workload, seed: int, g: int, t_prefix: int):
    """Group g's first t_prefix positions (inputs only; generation is not oracle work)."""
    t_prefix = min(t_prefix, w.T)
    gi = syn.group_inputs(w, seed, g, 1)
    rows = (np.arange(g * w.K, (g + 1) * w.K)[:, None] * w.T + np.arange(t_prefix)[None, :]).reshape(-1)
    lg = syn.logits_rows_f64_host(seed, w.V, rows, w.dtype).reshape(w.K, t_prefix, w.V)
    return lg, gi["tokens"][:, :t_prefix], gi["mask"][:, :t_prefix], gi["ref_logp"], gi["log_reward"]


def _oracle_group(w: syn.Workload, inputs):
    """The oracle as it stands (a1-a5, fwd + bwd) on one group's sample; returns valid tokens."""
    from oracle import tba_oracle as O
    lg, tok, mask, ref, rew = inputs
    O.vargrad_head(lg, tok, mask, ref, rew, w.beta, w.K, n_global=w.N)
    return int(mask.sum())


def _oracle_worker(i, inq, outq, barrier):
    sys.path.insert(0, ROOT)
    while True:
        job = inq.get()
        if job is None:
            return
        w, seed, g, tp = job
        inputs = _oracle_inputs(w, seed, g, tp)   # untimed
        barrier.wait()                            # every worker starts its oracle work together
        t0 = time.time()
        toks = _oracle_group(w, inputs)
        outq.put((i, t0, time.time(), toks))


class OraclePool:
    """P persistent worker processes (P = the host cores this process may use), one input queue
    each: per step every worker regenerates its own group's sample (untimed), all meet at a barrier,
    then run the oracle; the step's wall time is max(end) - min(start) over the workers."""

    def __init__(self, procs: int | None = None):
        import multiprocessing as mp
        ctx = mp.get_context("spawn")
        self.P = procs or max(1, len(os.sched_getaffinity(0)))
        self.barrier = ctx.Barrier(self.P)
        self.outq = ctx.Queue()
        self.inqs = [ctx.Queue() for _ in range(self.P)]
        self.procs = [ctx.Process(target=_oracle_worker, args=(i, self.inqs[i], self.outq, self.barrier), daemon=True)
                      for i in range(self.P)]
        for pr in self.procs:
            pr.start()

    def step(self, w: syn.Workload, seed: int, groups, tp: int):
        """Worker i takes group groups[i]; returns (wall seconds, valid tokens)."""
        for i in range(self.P):
            self.inqs[i].put((w, seed, int(groups[i]), tp))
        res = [self.outq.get(timeout=1800) for _ in range(self.P)]  # a dead worker raises, never hangs
        return max(r[2] for r in res) - min(r[1] for r in res), sum(r[3] for r in res)

    def close(self):
        for q in self.inqs:
            q.put(None)
        for pr in self.procs:
            pr.join(timeout=10)


def oracle_baseline(w: syn.Workload, tp: int, steps: int = 1, warmup: int = 0, pool: OraclePool | None = None):
    """The oracle on P host cores: every step, worker i runs global group i's first tp positions
    (a1-a5, fwd + bwd). Plus a single-core figure (one group, in this process). Returns a dict."""
    own = pool is None
    pool = pool or OraclePool()
    groups = list(range(pool.P))
    for _ in range(warmup):
        pool.step(w, SEED, groups, tp)
    secs, toks = 0.0, 0
    for _ in range(steps):
        s_, t_ = pool.step(w, SEED, groups, tp)
        secs += s_
        toks += t_
    if own:
        pool.close()
    inputs = _oracle_inputs(w, SEED, 0, tp)
    t0 = time.perf_counter()
    t1_toks = _oracle_group(w, inputs)
    t1 = time.perf_counter() - t0
    return {"value": toks / secs, "unit": "tokens/s", "cores": pool.P, "kind": "oracle", "cpu_model": cpu_model(),
            "sample": f"{pool.P} worker processes, worker i: global group i x K={w.K}, first {tp} positions "
                      f"({toks // max(steps, 1)} valid rows per step), oracle a1-a5 (fwd+bwd, fp64 NumPy) as it "
                      f"stands; {steps} step(s), {secs:.1f} s wall; input generation not timed",
            "single_core": {"value": t1_toks / t1, "unit": "tokens/s", "cores": 1,
                            "sample": f"group 0, first {tp} positions ({t1_toks} rows), one process, {t1:.1f} s"},
            "ms_per_step": secs / max(steps, 1) * 1e3}


def run_reference(args, w):
    """--impl reference: the fp64 oracle as it stands on all host cores, a bounded sample per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    tp = 16 if w.V * w.K > 200000 else 64
    cb = oracle_baseline(w, tp, steps=args.steps, warmup=args.warmup)
    line = {"impl": "reference", "metric": baseline_metric(), "value": cb["value"], "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "objective": args.objective, "note": w.note, "B_per_rank": w.B, "K": w.K,
                       "T": w.T, "V": w.V},
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "cpu_model", "sample",
                                                "single_core")},
            "e2e": {"value": cb["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- LM-head-fused arm (NEXT 3)
def tensor_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), \
            "measured (MEASURED_PEAKS.json bf16_tflops: cuBLAS 8192^3 burst; sustained beside it)"
    return 2250.0, 2250.0, "nominal dense bf16 (B200_PROFILING.md)"


def oracle_lmhead_sample(w: syn.Workload, n_rows: int, seed: int = SEED, chunk: int = 8192):
    """Bounded oracle sample for the LM-head arm: the first n_rows rows against the full
    vocabulary. Weight rows are generated chunk by chunk (not timed); the oracle's matmul +
    log-softmax is. Returns (seconds, rows)."""
    from oracle import tba_oracle as O
    tok, _ = syn.tokens_and_mask(w, seed, 0, max(1, -(-n_rows // w.T)))
    rows = np.arange(n_rows)
    h = syn.bf16_bits_to_f64(syn.hidden_rows(seed, w.d, rows))
    secs, zs = 0.0, []
    for v0 in range(0, w.V, chunk):
        wv = syn.bf16_bits_to_f64(syn.weight_rows(seed, w.d, np.arange(v0, min(w.V, v0 + chunk))))
        t0 = time.perf_counter()
        zs.append(O.lmhead_logits(h, wv))
        secs += time.perf_counter() - t0
    t0 = time.perf_counter()
    z = np.concatenate(zs, axis=1)
    for r in range(n_rows):
        O.token_logprob(z[r], int(tok.reshape(-1)[r]))
    secs += time.perf_counter() - t0
    return secs, n_rows


def lmhead_bench(args, w, tba, torch, dist, dev, world, rank, group):
    """One step = tba_lmhead_tb_loss_fwd over this rank's groups (z = W h on tcgen05 with the
    online log-softmax fused; Eq. 4/5 head), + the 24-byte all-reduce when N > 1."""
    B, K, T, V, d = w.B, w.K, w.T, w.V, w.d
    N = B * K
    g0 = rank * B
    n_global = float(N * world)
    gi = syn.group_inputs(w, SEED, g0, B)
    hidden = torch.empty((N, T, d), dtype=torch.bfloat16, device=dev)
    weight = torch.empty((V, d), dtype=torch.bfloat16, device=dev)
    syn.fill_bf16_cuda(hidden.view(N * T, d), SEED, "hidden", g0 * K * T)
    syn.fill_bf16_cuda(weight, SEED, "weight", 0)  # the model's LM head: replicated on every rank
    tokens = torch.from_numpy(gi["tokens"]).to(dev)
    mask = torch.from_numpy(gi["mask"]).to(dev)
    ref = torch.from_numpy(gi["ref_logp"]).to(dev)
    rew = torch.from_numpy(gi["log_reward"]).to(dev)
    ws = torch.empty(tba.lmhead_workspace_bytes(N, T, V), dtype=torch.uint8, device=dev)
    out = tba.ops._Fwd(N, K, dev)
    stream = torch.cuda.current_stream(dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def step():
        tba.lmhead_vargrad_fwd(hidden, weight, tokens, mask, ref, rew, w.beta, K, n_global, workspace=ws, out=out,
                               check_status=False)
        if group is not None:
            dist.all_reduce(out.partial, group=group)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if group is not None:
        dist.barrier()
    try:
        smi_id = "GPU-" + str(torch.cuda.get_device_properties(dev).uuid)
    except Exception:
        smi_id = str(dev.index)
    t0, t1 = ev(), ev()
    with Clocks(smi_id) as clk:
        torch.cuda.synchronize()
        if group is not None:
            dist.barrier()
        t0.record(stream)
        for _ in range(args.steps):
            step()
        t1.record(stream)
        torch.cuda.synchronize()
    ms = torch.tensor([t0.elapsed_time(t1) / args.steps], dtype=torch.float64, device=dev)
    if group is not None:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX, group=group)
    ms = ms.item()
    loss = out.partial[0].item()
    rows = N * T
    valid = int(gi["mask"].sum())

    # unfused comparison on the same inputs: cuBLAS writes the logits, then the logits-path forward.
    # Interleaved with the fused step (A B A B A B), because this load is power-capped and the
    # clock drifts with temperature: the medians of paired runs compare like with like.
    variants = {}
    if rank == 0 and world == 1 and not args.no_variants:
        logits = torch.empty((N, T, V), dtype=torch.bfloat16, device=dev)

        def unfused(mm_only=False):
            torch.matmul(hidden.view(rows, d), weight.T, out=logits.view(rows, V))
            if not mm_only:
                tba.vargrad_fwd(logits, tokens, mask, ref, rew, w.beta, K, n_global, check_status=False)

        def timed(fn, n):
            a, b = ev(), ev()
            torch.cuda.synchronize()
            a.record(stream)
            for _ in range(n):
                fn()
            b.record(stream)
            torch.cuda.synchronize()
            return a.elapsed_time(b) / n
        for _ in range(2):
            unfused()
        n = max(3, args.steps // 4)
        fz, uf, mm = [], [], []
        for _ in range(3):
            fz.append(timed(step, n))
            uf.append(timed(unfused, n))
            mm.append(timed(lambda: unfused(True), n))
        med = statistics.median
        variants["unfused_cublas_logits"] = {
            "ms_per_step": med(uf), "matmul_ms": med(mm), "fused_ms_paired": med(fz),
            "fused_over_unfused": med(fz) / med(uf), "value": valid / (med(uf) / 1e3), "unit": "tokens/s",
            "pairs": 3, "steps_per_run": n,
            "what": "torch.matmul (cuBLAS bf16) writes the [rows, V] logits, then tba_vargrad_tb_loss_fwd reads them; "
                    "timed interleaved with the fused step (medians)",
            "logits_bytes_written_and_read": rows * V * 2}
        del logits

    e2e = None
    if not args.no_e2e:
        h_hidden = torch.empty(hidden.shape, dtype=torch.bfloat16, pin_memory=True)
        h_hidden.copy_(hidden)
        h_tok, h_mask = tokens.cpu().pin_memory(), mask.cpu().pin_memory()
        h_ref, h_rew = ref.cpu().pin_memory(), rew.cpu().pin_memory()
        h_loss = torch.empty(1, dtype=torch.float64, pin_memory=True)
        h2d = sum(t.numel() * t.element_size() for t in (h_hidden, h_tok, h_mask, h_ref, h_rew))

        def e2e_step():
            hidden.copy_(h_hidden, non_blocking=True)
            tokens.copy_(h_tok, non_blocking=True)
            mask.copy_(h_mask, non_blocking=True)
            ref.copy_(h_ref, non_blocking=True)
            rew.copy_(h_rew, non_blocking=True)
            step()
            h_loss.copy_(out.partial[:1], non_blocking=True)
        e2e_step()
        torch.cuda.synchronize()
        a, b = ev(), ev()
        a.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        b.record(stream)
        torch.cuda.synchronize()
        e_ms = torch.tensor([a.elapsed_time(b) / args.e2e_steps], dtype=torch.float64, device=dev)
        if group is not None:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX, group=group)
        e_ms = e_ms.item()
        e2e = {"value": valid * world / (e_ms / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": 8, "ms_per_step": e_ms, "steps": args.e2e_steps,
               "path": "pinned host hidden states -> cudaMemcpyAsync -> tba_lmhead_tb_loss_fwd (C ABI) -> loss D2H; "
                       "the LM-head weight stays resident (a model parameter)"}
        assert abs(h_loss.item() - loss) <= 1e-12 * max(1.0, abs(loss))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        nr = 16
        secs, nrows = oracle_lmhead_sample(w, nr)
        cpu = {"value": nrows / secs, "unit": "tokens/s", "cores": int(os.environ.get("OMP_NUM_THREADS", "0")) or
               len(os.sched_getaffinity(0)), "kind": "oracle",
               "sample": f"first {nr} rows x full vocabulary: oracle z = W h (fp64 NumPy matmul, multithreaded BLAS) "
                         f"+ log-softmax, {secs:.1f} s (weight-row generation not timed)"}

    if rank == 0:
        peak, peak_sus, src = tensor_peak()
        flops = 2.0 * valid * V * d  # useful work: masked rows need no logits (whole masked row blocks are skipped)
        tf = flops / (ms / 1e3) / 1e12
        line = {
            "metric": baseline_metric() + " [LM-head-fused forward from hidden states, NEXT 3]",
            "value": valid * world / (ms / 1e3), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (tba_synth hidden states / LM-head weight, DESIGN.md §6)",
            "config": {"workload": w.name, "objective": "lmhead", "note": w.note, "B_per_rank": B, "K": K, "T": T,
                       "V": V, "d": d, "beta": w.beta, "rows_per_rank": rows,
                       "parallelism": f"group-sharded x{world}",
                       "l2": "weight 1.09 GB + hidden 0.47 GB per rank >> 126 MB L2; no flush needed"},
            "roofline": {"bound": "tensor", "kernel": "lmhead_fwd (+ lmhead_combine, seq_head in the same timing)",
                         "achieved": tf, "peak": peak, "unit": "TFLOP/s", "frac": tf / peak,
                         "frac_of_sustained_peak": tf / peak_sus, "peak_source": src,
                         "traffic": ncu_traffic(w.name, "lmhead_fwd"),
                         "algorithmic_flops_per_launch": flops, "avg_launch_ms": ms},
            "clocks": clk.summary(), "e2e": e2e, "cpu_baseline": cpu, "variants": variants,
            "gpu_launches": args.steps * 3,  # lmhead_fwd, lmhead_combine, seq_head
            "loss": loss,
        }
        print(json.dumps(line), flush=True)
    if group is not None:
        dist.barrier()
        dist.destroy_process_group()


def lmhead_train_bench(args, w, tba, torch, dist, dev, world, rank, group):
    """One step = the LM-head-fused forward AND backward over this rank's groups: tba_lmhead_tb_loss_fwd
    (z = W h on tcgen05, online log-softmax, Eq. 4/5 head) + the 24-byte all-reduce when N > 1 +
    tba_lmhead_tb_loss_bwd (dz recomputed tile by tile on tcgen05, dhidden = dZ W in bf16, dW = dZ^T H
    in fp32). The logits and dlogits never exist as [rows, V] tensors."""
    B, K, T, V, d = w.B, w.K, w.T, w.V, w.d
    N = B * K
    g0 = rank * B
    n_global = float(N * world)
    gi = syn.group_inputs(w, SEED, g0, B)
    hidden = torch.empty((N, T, d), dtype=torch.bfloat16, device=dev)
    weight = torch.empty((V, d), dtype=torch.bfloat16, device=dev)
    syn.fill_bf16_cuda(hidden.view(N * T, d), SEED, "hidden", g0 * K * T)
    syn.fill_bf16_cuda(weight, SEED, "weight", 0)
    tokens = torch.from_numpy(gi["tokens"]).to(dev)
    mask = torch.from_numpy(gi["mask"]).to(dev)
    ref = torch.from_numpy(gi["ref_logp"]).to(dev)
    rew = torch.from_numpy(gi["log_reward"]).to(dev)
    ws = torch.empty(tba.lmhead_workspace_bytes(N, T, V), dtype=torch.uint8, device=dev)
    bws = torch.empty(tba.lmhead_bwd_workspace_bytes(N, T, d, V, args.lm_chunk), dtype=torch.uint8, device=dev)
    out = tba.ops._Fwd(N, K, dev)
    dh = torch.empty((N, T, d), dtype=torch.bfloat16, device=dev)
    dw = torch.empty((V, d), dtype=torch.float32, device=dev)
    fb_ws = torch.empty(tba.lmhead_fwd_bwd_workspace_bytes(N, T, d, V, K, args.lm_groups), dtype=torch.uint8,
                        device=dev)
    stream = torch.cuda.current_stream(dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    marks = {}
    one_call = args.lm_schedule == "one-call"

    def step_one(rec=False):
        tba.lmhead_vargrad_fwd_bwd(hidden, weight, tokens, mask, ref, rew, w.beta, K, n_global, dhidden=dh,
                                   dweight=dw, groups_per_chunk=args.lm_groups, workspace=ws, bwd_workspace=fb_ws,
                                   out=out, check_status=False)
        if group is not None:
            dist.all_reduce(out.partial, group=group)

    def step_two(rec=False):
        if rec:
            marks["a"].record(stream)
        tba.lmhead_vargrad_fwd(hidden, weight, tokens, mask, ref, rew, w.beta, K, n_global, workspace=ws, out=out,
                               check_status=False)
        if group is not None:
            dist.all_reduce(out.partial, group=group)
        if rec:
            marks["b"].record(stream)
        tba.lmhead_vargrad_bwd(hidden, weight, tokens, mask, ws, out.resid, 2.0 / n_global, dhidden=dh, dweight=dw,
                               chunk_rows=args.lm_chunk, bwd_workspace=bws)
        if rec:
            marks["c"].record(stream)

    step = step_one if one_call else step_two
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if group is not None:
        dist.barrier()
    try:
        smi_id = "GPU-" + str(torch.cuda.get_device_properties(dev).uuid)
    except Exception:
        smi_id = str(dev.index)
    t0, t1 = ev(), ev()
    with Clocks(smi_id) as clk:
        torch.cuda.synchronize()
        if group is not None:
            dist.barrier()
        t0.record(stream)
        for _ in range(args.steps):
            step()
        t1.record(stream)
        torch.cuda.synchronize()
    ms = torch.tensor([t0.elapsed_time(t1) / args.steps], dtype=torch.float64, device=dev)
    if group is not None:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX, group=group)
    ms = ms.item()
    # phase split of the two-call schedule (one extra step with events between the calls)
    marks.update(a=ev(), b=ev(), c=ev())
    step_two(rec=True)
    torch.cuda.synchronize()
    fwd_ms, bwd_ms = marks["a"].elapsed_time(marks["b"]), marks["b"].elapsed_time(marks["c"])
    loss = out.partial[0].item()
    rows = N * T
    valid = int(gi["mask"].sum())

    variants = {}
    if rank == 0 and world == 1 and not args.no_variants:
        # unfused on the same inputs: cuBLAS logits -> logits-path fwd + bwd (dlogits in place) -> cuBLAS dH, dW
        logits = torch.empty((N, T, V), dtype=torch.bfloat16, device=dev)
        lws = torch.empty(tba.workspace_bytes(N, T), dtype=torch.uint8, device=dev)
        dh_u = torch.empty((rows, d), dtype=torch.bfloat16, device=dev)
        dw_u = torch.empty((V, d), dtype=torch.bfloat16, device=dev)

        def unfused():
            lg = logits.view(rows, V)
            torch.matmul(hidden.view(rows, d), weight.T, out=lg)
            o, _ = tba.vargrad_fwd(logits, tokens, mask, ref, rew, w.beta, K, n_global, workspace=lws,
                                   check_status=False)
            tba.vargrad_bwd(logits, tokens, mask, lws, o.resid, 2.0 / n_global, dlogits=logits)
            torch.matmul(lg, weight, out=dh_u)
            torch.matmul(lg.T, hidden.view(rows, d), out=dw_u)

        def timed(fn, n):
            a, b = ev(), ev()
            torch.cuda.synchronize()
            a.record(stream)
            for _ in range(n):
                fn()
            b.record(stream)
            torch.cuda.synchronize()
            return a.elapsed_time(b) / n
        unfused()
        other = step_two if one_call else step_one
        n = max(2, args.steps // 4)
        fz, uf, ot = [], [], []
        for _ in range(3):
            fz.append(timed(step, n))
            uf.append(timed(unfused, n))
            ot.append(timed(other, n))
        med = statistics.median
        variants["two_call" if one_call else "one_call"] = {
            "ms_per_step": med(ot), "ms_paired_this_schedule": med(fz), "value": valid / (med(ot) / 1e3),
            "unit": "tokens/s",
            "what": ("tba_lmhead_tb_loss_fwd + tba_lmhead_tb_loss_bwd (z recomputed by a 4th GEMM)" if one_call else
                     "tba_lmhead_tb_loss_fwd_bwd (chunks of whole groups, logits stored in fp32 once)")}
        variants["unfused_cublas"] = {
            "ms_per_step": med(uf), "fused_ms_paired": med(fz), "fused_over_unfused": med(fz) / med(uf),
            "value": valid / (med(uf) / 1e3), "unit": "tokens/s", "pairs": 3, "steps_per_run": n,
            "what": "torch.matmul (cuBLAS bf16) writes the [rows, V] logits; tba_vargrad_tb_loss_fwd/_bwd (dlogits "
                    "in place, bf16); torch.matmul dH = dZ W and dW = dZ^T H (bf16 outputs); interleaved medians",
            "extra_hbm_bytes": rows * V * 2 * 2}
        del logits, lws, dh_u, dw_u

    if rank == 0:
        peak, peak_sus, src = tensor_peak()
        gemm = 2.0 * valid * V * d
        flops = 3 * gemm       # algorithmic: z = W h, dH = dZ W, dW = dZ^T H
        tf = flops / (ms / 1e3) / 1e12
        line = {
            "metric": baseline_metric() + " [LM-head-fused forward + backward from hidden states, NEXT 3]",
            "value": valid * world / (ms / 1e3), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (tba_synth hidden states / LM-head weight, DESIGN.md §6)",
            "config": {"workload": w.name, "objective": "lmhead_train", "note": w.note, "B_per_rank": B, "K": K,
                       "T": T, "V": V, "d": d, "beta": w.beta, "rows_per_rank": rows, "schedule": args.lm_schedule,
                       "groups_per_chunk": args.lm_groups, "chunk_rows": args.lm_chunk,
                       "dhidden_dtype": "bf16", "dweight_dtype": "fp32", "parallelism": f"group-sharded x{world}",
                       "l2": "weight 1.09 GB + hidden 0.47 GB + dz chunks per rank >> 126 MB L2; no flush needed"},
            "roofline": {"bound": "tensor", "kernel": "whole step (lmhead_fwd, 2x tc_gemm<STORE>, dz pass / "
                                                      "tc_gemm<DZ>, gathers, combine, head)",
                         "achieved": tf, "peak": peak, "unit": "TFLOP/s", "frac": tf / peak,
                         "frac_of_sustained_peak": tf / peak_sus, "peak_source": src,
                         "traffic": None, "algorithmic_flops_per_launch": flops, "avg_launch_ms": ms,
                         "executed_flops": (3 if one_call else 4) * gemm,
                         "note": "algorithmic = 3 GEMMs; the one-call schedule stores z (fp32, per chunk of whole "
                                 "groups), the two-call backward recomputes it (a 4th GEMM)"},
            "kernels": {"two_call_fwd_ms": fwd_ms, "two_call_bwd_ms": bwd_ms},
            "clocks": clk.summary(), "e2e": None, "cpu_baseline": None, "variants": variants,
            # one-call: per step W^T gather, tb_finish; per chunk lm_compact_units, lmhead_fwd, lmhead_combine,
            # seq_head, lmb_compact_rows, H gather, lmb_dz_from_z, tc_gemm<STORE> x2. Two-call: per step
            # lm_compact_units, lmhead_fwd, lmhead_combine, seq_head, lmb_compact_rows, W^T gather; per chunk
            # H gather, tc_gemm<DZ>, tc_gemm<STORE> x2 (cudaMemset launches not counted)
            "gpu_launches": args.steps * (
                (2 + 9 * -(-B // (args.lm_groups if args.lm_groups > 0 else max(1, 16384 // (K * T))))) if one_call
                else (6 + 4 * -(-rows // (args.lm_chunk if args.lm_chunk > 0 else 16384)))),
            "loss": loss,
        }
        print(json.dumps(line), flush=True)
    if group is not None:
        dist.barrier()
        dist.destroy_process_group()


# ----------------------------------------------------------------------------- strong scaling
def strong_bench(args, w, tba, torch, dist, dev, world, rank, group, local):
    """--scaling strong: the WHOLE global batch of `w` (e.g. qwen: 64 groups x K=8 x
    T=1024) at every N. Rank r takes a contiguous range of whole groups (dist.group_range; for ragged
    masks dist.token_balanced_ranges over the groups' valid-token counts) and streams it in chunks of
    --chunk-groups: per chunk tba_vargrad_tb_loss_fwd + _bwd with the GLOBAL normaliser 512 (Eq. 5's
    1/(BK)), through one resident chunk-sized logits buffer and one dlogits buffer (the whole
    batch's 160 GB of logits plus its dlogits do not fit one GPU). Every chunk reads the same resident
    logits (the rank's first chunk); its tokens, masks, references and rewards are its own. The chunk
    partials are all-reduced once per step on a side stream."""
    K, T, V = w.K, w.T, w.V
    Bg = w.B
    Ng = Bg * K
    _, mask_all = syn.tokens_and_mask(w, SEED, 0, Ng)
    gtok = mask_all.reshape(Bg, K * T).sum(1)
    if w.len_lo != w.len_hi:
        ranges = tba.token_balanced_ranges([int(x) for x in gtok], world)
        split = "token-balanced (dist.token_balanced_ranges)"
    else:
        ranges = [tba.group_range(Bg, world, r) for r in range(world)]
        split = "equal whole-group blocks (dist.group_range)"
    g_lo, g_hi = ranges[rank]
    cg = max(1, min(args.chunk_groups, Bg))
    chunks = [(g, min(g + cg, g_hi)) for g in range(g_lo, g_hi, cg)]
    dt = torch.bfloat16 if w.dtype == "bf16" else torch.float32
    esz = 2 if w.dtype == "bf16" else 4
    Nc = cg * K
    logits = torch.empty((Nc, T, V), dtype=dt, device=dev)
    syn.fill_logits_cuda(logits, SEED, (g_lo if chunks else 0) * K * T, V)
    dlogits = torch.empty_like(logits)
    ws = torch.empty(tba.workspace_bytes(Nc, T), dtype=torch.uint8, device=dev)
    partials = torch.zeros((max(len(chunks), 1), 3), dtype=torch.float64, device=dev)
    ins, outs = [], []
    for c, (a, b) in enumerate(chunks):
        gi = syn.group_inputs(w, SEED, a, b - a)
        ins.append([torch.from_numpy(gi[k]).to(dev) for k in ("tokens", "mask", "ref_logp", "log_reward")])
        o = tba.ops._Fwd((b - a) * K, K, dev)
        o.partial = partials[c]
        outs.append(o)
    valid_rank = int(gtok[g_lo:g_hi].sum())
    masked_rank = (g_hi - g_lo) * K * T - valid_rank
    stream = torch.cuda.current_stream(dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    pending = []

    def step(rec=None):
        for c, (a, b) in enumerate(chunks):
            n = (b - a) * K
            tok, msk, ref, rew = ins[c]
            tba.vargrad_fwd(logits[:n], tok, msk, ref, rew, w.beta, K, float(Ng), workspace=ws, out=outs[c],
                            check_status=False)
            if rec is not None:
                rec[c][0].record(stream)
            tba.vargrad_bwd(logits[:n], tok, msk, ws, outs[c].resid, 2.0 / Ng, dlogits=dlogits[:n])
            if rec is not None:
                rec[c][1].record(stream)
        if group is not None:
            pending.append(tba.allreduce_partial_async(partials, group))
            pending.pop().wait()  # before the next step rewrites the partials (the writers did not wait)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if group is not None:
        dist.barrier()
    recs = [[[ev(), ev()] for _ in chunks] for _ in range(args.steps)]
    t0, t1 = ev(), ev()
    try:
        smi_id = "GPU-" + str(torch.cuda.get_device_properties(dev).uuid)
    except Exception:
        smi_id = str(local)
    with Clocks(smi_id) as clk:
        torch.cuda.synchronize()
        if group is not None:
            dist.barrier()
        t0.record(stream)
        for i in range(args.steps):
            step(recs[i])
        t1.record(stream)
        torch.cuda.synchronize()
        if group is not None:
            dist.barrier()
    bwd_ms = sum(r[0].elapsed_time(r[1]) for rr in recs for r in rr) / args.steps
    tm = torch.tensor([t0.elapsed_time(t1) / args.steps, bwd_ms], dtype=torch.float64, device=dev)
    if group is not None:
        dist.all_reduce(tm, op=dist.ReduceOp.MAX, group=group)
    ms_step, bwd_ms = tm.tolist()
    glob = partials.clone()
    if group is not None:
        dist.all_reduce(glob, group=group)
    loss = float(glob[:, 0].sum().item())
    if rank == 0:
        peak, peak_src = peaks()
        bwd_bytes = valid_rank * V * 2 * esz + masked_rank * V * esz
        bwd_gbs = bwd_bytes / (bwd_ms / 1e3) / 1e9 if bwd_ms > 0 else None
        step_bytes = valid_rank * V * 3 * esz + masked_rank * V * esz
        line = {
            "metric": baseline_metric(), "value": int(gtok.sum()) / (ms_step / 1e3), "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": w.dtype,
            "data": "synthetic (tba_synth seeded generator, DESIGN.md §6)",
            "config": {"workload": w.name, "objective": "vargrad", "schedule": "two-call per chunk", "scaling": "strong",
                       "note": w.note, "B_global": Bg, "K": K, "T": T, "V": V, "beta": w.beta,
                       "groups_rank0": [g_lo, g_hi], "chunk_groups": cg, "chunks_rank0": len(chunks),
                       "split": split, "valid_tokens_global": int(gtok.sum()),
                       "parallelism": f"group-sharded x{world}",
                       "collective": "NCCL all_reduce of the chunk partials on a side stream" if world > 1 else None,
                       "logits_buffer": "one resident chunk buffer (rank's first chunk) read by every chunk; "
                                        "per-chunk tokens/masks/references/rewards are the chunk's own",
                       "l2": "chunk buffers (%.1f GB logits + dlogits) >> 126 MB L2; no flush needed" %
                             (logits.numel() * esz * 2 / 1e9)},
            "hbm_gbs_step_rank0": step_bytes / (ms_step / 1e3) / 1e9,
            "roofline": {"bound": "hbm", "kernel": "row_bwd (a5), summed over the rank's chunks", "achieved": bwd_gbs,
                         "peak": peak, "unit": "GB/s", "frac": (bwd_gbs / peak) if bwd_gbs else None,
                         "traffic": None, "algorithmic_bytes_per_launch": bwd_bytes / max(len(chunks), 1),
                         "avg_launch_ms": bwd_ms / max(len(chunks), 1), "peak_source": peak_src},
            "clocks": clk.summary(),
            "e2e": None, "cpu_baseline": None,
            "gpu_launches": args.steps * 3 * len(chunks),
            "loss": loss,
        }
        print(json.dumps(line), flush=True)
    if group is not None:
        dist.barrier()
        dist.destroy_process_group()


# ----------------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="qwen_shard", choices=sorted(syn.WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-variants", action="store_true", help="skip the deferred-scale variant measurement")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--schedule", default="two-call", choices=["two-call", "fused", "deferred", "pipelined"],
                    help="two-call: tba_vargrad_tb_loss_fwd + _bwd (3 kernels); fused: tba_tb_loss_fused (1 kernel); "
                         "deferred: tba_tb_loss_fwd_deferred (unscaled gradient, 4V bytes; NEXT 2 (ii)); "
                         "pipelined: tba_tb_loss_pipelined (group chunks, writer of chunk c-1 beside the forward "
                         "of chunk c on a second stream)")
    ap.add_argument("--pipe-one-stream", action="store_true",
                    help="--schedule pipelined on ONE stream (chunk kernels PDL-chained) instead of two")
    ap.add_argument("--pipe-groups", type=int, default=0,
                    help="groups per chunk for --schedule pipelined (0 = ~L2/4 of logits per chunk)")
    ap.add_argument("--cuda-graph", action="store_true",
                    help="replay the step's library calls from CUDA graphs (forward and backward captured separately)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: every rank owns --workload's B groups (rank r: groups [rB, rB+B)); strong: the "
                         "global batch of --workload (e.g. qwen: 64 x 8) split by whole groups over the N ranks "
                         "(token-balanced for ragged masks), each rank streaming its groups in chunks of "
                         "--chunk-groups through one resident chunk buffer (SURVEY §8(d))")
    ap.add_argument("--chunk-groups", type=int, default=8,
                    help="--scaling strong: groups per chunk (8 Qwen groups = 20 GB of logits + 20 GB of dlogits)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo + --share-gpu only to test the multi-rank flow on 1 GPU)")
    ap.add_argument("--share-gpu", action="store_true")
    ap.add_argument("--lm-chunk", type=int, default=0, help="rows per chunk of the LM-head backward (0 = 16384)")
    ap.add_argument("--lm-groups", type=int, default=0,
                    help="groups per chunk of the one-call LM-head fwd+bwd (0 = as many as fit 16384 rows)")
    ap.add_argument("--lm-schedule", default="one-call", choices=["one-call", "two-call"],
                    help="lmhead_train: tba_lmhead_tb_loss_fwd_bwd, or tba_lmhead_tb_loss_fwd + _bwd")
    ap.add_argument("--objective", default="vargrad", choices=["vargrad", "tbap", "lmhead", "lmhead_train"],
                    help="vargrad: Eq. 5 (the north-star head); tbap: the TBA' token-level rule (Eq. 16); "
                         "lmhead: the Eq. 4/5 forward from hidden states with the LM head fused (NEXT 3); "
                         "lmhead_train: that forward + the backward through the head (dhidden, dW)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    w = syn.WORKLOADS[args.workload]
    if args.impl == "reference":
        return run_reference(args, w)

    import torch
    import torch.distributed as dist

    import paper_2503_18929_b200 as tba

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.share_gpu:  # test mode: all ranks on cuda:0 (needs --dist-backend gloo; NCCL rejects duplicates)
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)
        group = dist.group.WORLD
    tba.load_library()
    if args.objective == "lmhead":
        return lmhead_bench(args, w, tba, torch, dist, dev, world, rank, group)
    if args.objective == "lmhead_train":
        return lmhead_train_bench(args, w, tba, torch, dist, dev, world, rank, group)
    if args.scaling == "strong":
        return strong_bench(args, w, tba, torch, dist, dev, world, rank, group, local)

    # ---- inputs: this rank's whole groups of the global batch, resident in HBM
    B, K, T, V = w.B, w.K, w.T, w.V
    N = B * K
    g0 = rank * B
    n_global = float(N * world)
    gi = syn.group_inputs(w, SEED, g0, B)
    dt = torch.bfloat16 if w.dtype == "bf16" else torch.float32
    logits = torch.empty((N, T, V), dtype=dt, device=dev)
    syn.fill_logits_cuda(logits, SEED, g0 * K * T, V)
    tokens = torch.from_numpy(gi["tokens"]).to(dev)
    mask = torch.from_numpy(gi["mask"]).to(dev)
    ref = torch.from_numpy(gi["ref_logp"]).to(dev)
    rew = torch.from_numpy(gi["log_reward"]).to(dev)
    dlogits = torch.empty_like(logits)
    ws = torch.empty(tba.workspace_bytes(N, T), dtype=torch.uint8, device=dev)
    tbap = args.objective == "tbap"
    out = tba.ops._TbapFwd(N, T, dev) if tbap else tba.ops._Fwd(N, K, dev)
    gen = torch.from_numpy(syn.gen_logp(w, SEED, g0 * K, N)).to(dev) if tbap else None
    n_tok_global = float(int(gi["mask"].sum()) * world)
    stream = torch.cuda.current_stream(dev)

    valid_rows = int(gi["mask"].sum())
    masked_rows = N * T - valid_rows
    esz = 2 if w.dtype == "bf16" else 4
    fwd_bytes = valid_rows * V * esz                              # a1 reads each valid row once
    bwd_bytes = valid_rows * V * 2 * esz + masked_rows * V * esz  # a5 reads+writes valid rows, zero-fills masked
    tokens_per_step_rank = valid_rows

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    pipelined = args.schedule == "pipelined"
    fused = args.schedule == "fused" or pipelined  # one call per step (fwd + bwd)
    deferred = args.schedule == "deferred"
    if (fused or deferred) and tbap:
        raise SystemExit("--schedule fused/pipelined/deferred implement the TB objectives (Eq. 5 / Eq. 3) only")
    gpc = args.pipe_groups if args.pipe_groups > 0 else int(os.environ.get("TBA_PIPE_GROUPS", "0"))
    if gpc <= 0:
        gpc = int(0.25 * torch.cuda.get_device_properties(dev).L2_cache_size // max(1, K * T * V * esz))
    gpc = max(1, min(B, gpc))
    n_chunks = -(-B // gpc)

    def fwd_call():
        if pipelined:
            tba.vargrad_pipelined(logits, tokens, mask, ref, rew, w.beta, K, n_global, workspace=ws, out=out,
                                  dlogits=dlogits, groups_per_chunk=gpc, check_status=False,
                                  aux_stream=not args.pipe_one_stream)
        elif fused:
            tba.vargrad_fused(logits, tokens, mask, ref, rew, w.beta, K, n_global, workspace=ws, out=out,
                              dlogits=dlogits, check_status=False)
        elif deferred:
            tba.vargrad_fwd_deferred(logits, tokens, mask, ref, rew, w.beta, K, n_global, workspace=ws, out=out,
                                     grad_unscaled=dlogits, check_status=False)
        elif tbap:
            tba.tbap_fwd(logits, tokens, mask, gen, ref, rew, w.beta, K, "clip", 0.0, 8.0, n_tok_global,
                         workspace=ws, out=out, check_status=False)
        else:
            tba.vargrad_fwd(logits, tokens, mask, ref, rew, w.beta, K, n_global, workspace=ws, out=out,
                            check_status=False)

    def bwd_call():
        if fused or deferred:
            pass
        elif tbap:
            tba.tbap_bwd(logits, tokens, mask, ws, out.coef, n_tok_global, dlogits=dlogits)
        else:
            tba.vargrad_bwd(logits, tokens, mask, ws, out.resid, 2.0 / n_global, dlogits=dlogits)

    if args.cuda_graph:
        g_fwd, g_bwd = tba.CapturedStep(fwd_call), tba.CapturedStep(bwd_call)
        run_fwd, run_bwd = g_fwd.replay, g_bwd.replay
    else:
        run_fwd, run_bwd = fwd_call, bwd_call

    pending = []

    def step(rec=None):
        # The 24-byte partials all-reduce runs on a side stream (tba.allreduce_partial_async): the
        # gradient writer does not wait for it (N_global is static); the next step's forward, which
        # rewrites the partials, waits for it.
        if rec is not None:
            rec[0].record(stream)
        run_fwd()
        if rec is not None:
            rec[1].record(stream)
        if group is not None:
            pending.append(tba.allreduce_partial_async(out.partial, group))
        if rec is not None:
            rec[2].record(stream)
        run_bwd()
        if rec is not None:
            rec[3].record(stream)
        if pending:
            pending.pop().wait()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if group is not None:
        dist.barrier()
    recs = [[ev() for _ in range(4)] for _ in range(args.steps)]
    t0, t1 = ev(), ev()
    try:
        smi_id = "GPU-" + str(torch.cuda.get_device_properties(dev).uuid)
    except Exception:
        smi_id = str(local)
    with Clocks(smi_id) as clk:
        torch.cuda.synchronize()
        if group is not None:
            dist.barrier()
        t0.record(stream)
        for i in range(args.steps):
            step(recs[i])
        t1.record(stream)
        torch.cuda.synchronize()
        if group is not None:
            dist.barrier()
    ms_total = t0.elapsed_time(t1)
    fwd_ms = statistics.mean(r[0].elapsed_time(r[1]) for r in recs)
    bwd_ms = statistics.mean(r[2].elapsed_time(r[3]) for r in recs)
    ms_step = ms_total / args.steps
    tmax = torch.tensor([ms_step, fwd_ms, bwd_ms], dtype=torch.float64, device=dev)
    if group is not None:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX, group=group)
    ms_step, fwd_ms, bwd_ms = tmax.tolist()
    loss = out.partial[0].item()
    if group is not None:  # the step's global loss (the side-stream all-reduce of the last step)
        g_ = out.partial.clone()
        dist.all_reduce(g_, group=group)
        loss = g_[0].item()

    # ---- variant: the deferred-scale schedule on the same inputs
    variants = {}
    if not (fused or deferred or tbap) and not args.no_variants:
        def dstep():
            tba.vargrad_fwd_deferred(logits, tokens, mask, ref, rew, w.beta, K, n_global, workspace=ws, out=out,
                                     grad_unscaled=dlogits, check_status=False)
            if group is not None:
                dist.all_reduce(out.partial, group=group)
        for _ in range(args.warmup):
            dstep()
        torch.cuda.synchronize()
        if group is not None:
            dist.barrier()
        a, b = ev(), ev()
        a.record(stream)
        for _ in range(args.steps):
            dstep()
        b.record(stream)
        torch.cuda.synchronize()
        d_ms = torch.tensor([a.elapsed_time(b) / args.steps], dtype=torch.float64, device=dev)
        if group is not None:
            dist.all_reduce(d_ms, op=dist.ReduceOp.MAX, group=group)
        d_ms = d_ms.item()
        variants["deferred_scale"] = {
            "ms_per_step": d_ms, "value": tokens_per_step_rank * world / (d_ms / 1e3), "unit": "tokens/s",
            "what": "tba_tb_loss_fwd_deferred: loss + UNSCALED gradient G in one pass per row; "
                    "dlogits = (2/N) eps_s G is applied by the consumer (DESIGN.md §5.4)",
            "gpu_launches_per_step": 2}

    # ---- e2e: the same step through the public API from pinned HOST buffers
    e2e = None
    if not args.no_e2e:
        # Host memory guard: every local rank pins its whole per-step input. If the box cannot
        # hold that for all local ranks (e.g. 8 x 20 GB on a 196 GB host), the e2e step runs on
        # the leading groups that fit and says so (same metric, smaller step).
        import psutil
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
        per_group = K * T * V * esz + K * T * 9 + K * 16 + (K * T * 4 if tbap else 0)
        budget = 0.6 * psutil.virtual_memory().available / max(local_world, 1)
        ge = int(max(1, min(B, budget // per_group)))
        nk = ge * K
        lg_e, tok_e, mask_e, ref_e, rew_e = logits[:nk], tokens[:nk], mask[:nk], ref[:nk], rew[:nk]
        gen_e = gen[:nk] if tbap else None
        h_logits = torch.empty(lg_e.shape, dtype=dt, pin_memory=True)
        h_logits.copy_(lg_e)
        h_tok = tok_e.cpu().pin_memory()
        h_mask = mask_e.cpu().pin_memory()
        h_ref = ref_e.cpu().pin_memory()
        h_rew = rew_e.cpu().pin_memory()
        h_gen = gen_e.cpu().pin_memory() if tbap else None
        h_loss = torch.empty(1, dtype=torch.float64, pin_memory=True)
        h2d = sum(t.numel() * t.element_size() for t in (h_logits, h_tok, h_mask, h_ref, h_rew)
                  + ((h_gen,) if tbap else ()))
        ng_e = float(nk * world)
        ntok_e = float(int(h_mask.sum()) * world)
        valid_e = int(h_mask.sum())

        def e2e_step():
            lg_e.copy_(h_logits, non_blocking=True)
            tok_e.copy_(h_tok, non_blocking=True)
            mask_e.copy_(h_mask, non_blocking=True)
            ref_e.copy_(h_ref, non_blocking=True)
            rew_e.copy_(h_rew, non_blocking=True)
            if deferred:
                tba.vargrad_fwd_deferred(lg_e, tok_e, mask_e, ref_e, rew_e, w.beta, K, ng_e, workspace=ws, out=out,
                                         grad_unscaled=dlogits[:nk], check_status=False)
                if group is not None:
                    dist.all_reduce(out.partial, group=group)
                h_loss.copy_(out.partial[:1], non_blocking=True)
                return
            if pipelined:
                tba.vargrad_pipelined(lg_e, tok_e, mask_e, ref_e, rew_e, w.beta, K, ng_e, workspace=ws, out=out,
                                      dlogits=dlogits[:nk], groups_per_chunk=gpc, check_status=False)
                if group is not None:
                    dist.all_reduce(out.partial, group=group)
                h_loss.copy_(out.partial[:1], non_blocking=True)
                return
            if fused:
                tba.vargrad_fused(lg_e, tok_e, mask_e, ref_e, rew_e, w.beta, K, ng_e, workspace=ws, out=out,
                                  dlogits=dlogits[:nk], check_status=False)
                if group is not None:
                    dist.all_reduce(out.partial, group=group)
                h_loss.copy_(out.partial[:1], non_blocking=True)
                return
            if tbap:
                gen_e.copy_(h_gen, non_blocking=True)
                tba.tbap_fwd(lg_e, tok_e, mask_e, gen_e, ref_e, rew_e, w.beta, K, "clip", 0.0, 8.0, ntok_e,
                             workspace=ws, out=out, check_status=False)
            else:
                tba.vargrad_fwd(lg_e, tok_e, mask_e, ref_e, rew_e, w.beta, K, ng_e, workspace=ws, out=out,
                                check_status=False)
            if group is not None:
                dist.all_reduce(out.partial, group=group)
            if tbap:
                tba.tbap_bwd(lg_e, tok_e, mask_e, ws, out.coef, ntok_e, dlogits=dlogits[:nk])
            else:
                tba.vargrad_bwd(lg_e, tok_e, mask_e, ws, out.resid, 2.0 / ng_e, dlogits=dlogits[:nk])
            h_loss.copy_(out.partial[:1], non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        if group is not None:
            dist.barrier()
        a, b = ev(), ev()
        a.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        b.record(stream)
        torch.cuda.synchronize()
        e_ms = torch.tensor([a.elapsed_time(b) / args.e2e_steps], dtype=torch.float64, device=dev)
        if group is not None:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX, group=group)
        e_ms = e_ms.item()
        e2e = {"value": valid_e * world / (e_ms / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 8, "ms_per_step": e_ms, "steps": args.e2e_steps,
               "path": "pinned host -> cudaMemcpyAsync -> libtba fwd/bwd (C ABI) -> loss D2H",
               "groups_per_rank": ge}
        if ge < B:
            e2e["note"] = (f"host RAM holds pinned inputs for {ge} of {B} groups per rank x {local_world} local "
                           f"ranks; e2e step = those groups")
        elif not tbap:
            assert abs(h_loss.item() - loss) <= 1e-12 * max(1.0, abs(loss))
        del h_logits

    # ---- cpu baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_baseline(w, 128 if w.V * K > 200000 else 256)
        cpu.pop("ms_per_step", None)

    if rank == 0:
        peak, peak_src = peaks()
        bwd_gbs = bwd_bytes / (bwd_ms / 1e3) / 1e9 if bwd_ms > 0 else None
        fwd_gbs = fwd_bytes / (fwd_ms / 1e3) / 1e9
        step_gbs = (fwd_bytes + bwd_bytes) / (ms_step / 1e3) / 1e9
        if fused or deferred:
            # one kernel; its unique bytes are 2V read + 2V write per valid row (+2V zero-fill per masked
            # row): the backward re-read is served by L2 when the lookahead window fits
            fused_bytes = valid_rows * V * 2 * esz + masked_rows * V * esz
            fgbs = fused_bytes / (fwd_ms / 1e3) / 1e9
            kname = ("row_single (deferred scale)" if deferred else
                     f"pipelined step (row_fwd_rows + seq_head + row_bwd per chunk of {gpc} groups)" if pipelined
                     else "tb_fused (a1-a5 in one launch)")
            roof = {"bound": "hbm", "kernel": kname, "achieved": fgbs, "peak": peak,
                    "unit": "GB/s", "frac": fgbs / peak, "traffic": ncu_traffic(w.name, "row_single" if deferred else "pipelined" if pipelined else "tb_fused"),
                    "algorithmic_bytes_per_launch": fused_bytes, "avg_launch_ms": fwd_ms, "peak_source": peak_src,
                    "bytes_model": "4V per valid token (unique); the two-pass schedule's 6V is in hbm_gbs_step"}
            kern = {"fused_ms": fwd_ms, "fused_unique_gbs": fgbs}
        else:
            tr = ncu_traffic(w.name, "row_bwd")
            roof = {"bound": "hbm", "kernel": "row_bwd (a5, dominant: 2/3 of bytes)", "achieved": bwd_gbs,
                    "peak": peak, "unit": "GB/s", "frac": bwd_gbs / peak, "traffic": tr,
                    "algorithmic_bytes_per_launch": bwd_bytes, "avg_launch_ms": bwd_ms, "peak_source": peak_src,
                    "frac_of_nominal": bwd_gbs / NOMINAL_HBM_GBS, "nominal_peak": NOMINAL_HBM_GBS}
            kern = {"fwd_ms": fwd_ms, "fwd_gbs": fwd_gbs, "fwd_frac": fwd_gbs / peak, "bwd_ms": bwd_ms,
                    "bwd_gbs": bwd_gbs, "step_frac": step_gbs / peak,
                    "fwd_frac_of_nominal": fwd_gbs / NOMINAL_HBM_GBS, "step_frac_of_nominal": step_gbs / NOMINAL_HBM_GBS,
                    "note": "frac = of the measured copy bandwidth (MEASURED_PEAKS hbm_gbs, read+write); a read-only "
                            "kernel (the forward) can exceed it: its own read-only ceiling is ~7.0-7.3 TB/s "
                            "(scripts/microbench); frac_of_nominal = of the 7.7 TB/s HGX figure"}
        line = {
            "metric": baseline_metric() + (" [TBA' Eq. 16 objective]" if tbap else ""),
            "value": tokens_per_step_rank * world / (ms_step / 1e3),
            "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": w.dtype, "data": "synthetic (tba_synth seeded generator, DESIGN.md §6)",
            "config": {"workload": w.name, "objective": args.objective, "schedule": args.schedule, "scaling": "weak",
                       **({"groups_per_chunk": gpc, "chunks": n_chunks,
                           "streams": 1 if args.pipe_one_stream else 2} if pipelined else {}),
                       "cuda_graph": bool(args.cuda_graph), "note": w.note,
                       "B_per_rank": B, "B_global": B * world, "K": K, "T": T,
                       "V": V, "beta": w.beta, "logits_dtype": w.dtype, "dlogits_dtype": w.dtype,
                       "valid_tokens_per_rank": valid_rows, "parallelism": f"group-sharded x{world}",
                       "collective": ("NCCL all_reduce of 24 B on a side stream, overlapped with row_bwd"
                                      if world > 1 else None),
                       "l2": "inputs (%.1f GB logits + dlogits per rank) >> 126 MB L2; no flush needed" %
                             ((logits.numel() * esz * 2) / 1e9)},
            "hbm_gbs_step": step_gbs,
            "roofline": roof,
            "kernels": kern,
            "clocks": clk.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
            "variants": variants,
            # our kernels per step: pipelined 3 per chunk + the finisher; fused 1; deferred row_single + seq_head;
            # two-call row_fwd_rows + seq_head (tbap_head) + row_bwd
            "gpu_launches": args.steps * ((3 * n_chunks + 1) if pipelined else 1 if fused else 2 if deferred else 3),
            "loss": loss,
        }
        print(json.dumps(line), flush=True)
    if group is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
