"""The loss all-reduce fused into the head kernel over peer memory (tba_tb_loss_fwd_peer), run by
two processes on one GPU (CUDA IPC between processes works on a single device too): both ranks
get the global loss bit-identically, equal to the sum of the separately computed shard partials,
over several epochs; a missing peer times out instead of hanging."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import dataclasses
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    import paper_2503_18929_b200 as tba
    import tba_synth as syn
    from tests import _harness as H
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    w = dataclasses.replace(syn.WORKLOADS["pythia"], B=6, K=4, T=5)
    g0, g1 = tba.group_range(w.B, world, rank)
    inp = H.device_inputs(w, 3, g0, g1 - g0)
    N = w.N
    pr = tba.PeerReducer(dist.group.WORLD, "cuda:0", timeout_s=30.0)
    results = []
    for epoch in range(3):
        o, _ = tba.vargrad_fwd(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"],
                               w.beta, w.K, float(N), peer=pr, check_status=True)
        ref, _ = tba.vargrad_fwd(inp["logits"], inp["tokens"], inp["mask"], inp["ref_logp"], inp["log_reward"],
                                 w.beta, w.K, float(N))
        torch.cuda.synchronize()
        local = ref.partial.cpu()
        tot = local.clone()
        dist.all_reduce(tot)  # gloo on CPU: the reference sum
        results.append((o.partial.cpu().numpy().tobytes(), tot.numpy()))
    allres = [None] * world
    dist.all_gather_object(allres, [r[0] for r in results])
    pr.close()
    q.put((rank, results, allres))
    dist.barrier()
    dist.destroy_process_group()


def test_fused_peer_allreduce_two_processes_one_gpu():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, results, allres in out:
        for e, (peer_bytes, ref_tot) in enumerate(results):
            got = np.frombuffer(peer_bytes, dtype=np.float64)
            assert abs(got[0] - ref_tot[0]) <= 1e-12 * abs(ref_tot[0]) and got[1] == ref_tot[1] and got[2] == ref_tot[2]
            assert allres[0][e] == allres[1][e]  # bit-identical on both ranks


def test_peer_args_validation():
    import ctypes

    from paper_2503_18929_b200 import _lib
    from paper_2503_18929_b200._lib import TbaPeerReduce, TbaRows
    L = _lib.load()
    x = TbaRows(0x10000, 0, 0, 4, 2, 8, 8, 0x10000, 0x10000)
    for pr in (TbaPeerReduce(0, 0x1000, 0, 2, 1, 1.0), TbaPeerReduce(0x1000, 0x1000, 2, 2, 1, 1.0),
               TbaPeerReduce(0x1000, 0x1000, 0, 2, 0, 1.0), TbaPeerReduce(0x1000, 0x1000, 0, 2, 1, 0.0)):
        rc = L.tba_tb_loss_fwd_peer(ctypes.byref(x), None, 0x1000, 0x1000, 1.0, 2, 4.0, 0x100000, 0x1000, 0x1000,
                                    0x1000, 0x1000, 0x1000, ctypes.byref(pr), None, None)
        assert rc == _lib.TBA_ERR_INVALID_ARG


def test_missing_peer_times_out_instead_of_hanging():
    import ctypes
    import dataclasses

    import paper_2503_18929_b200 as tba
    import tba_synth as syn
    from paper_2503_18929_b200 import _lib
    from paper_2503_18929_b200._lib import TbaPeerReduce
    from tests import _harness as H
    L = _lib.load()
    bufs = []
    for nbytes in (2 * 2 * 4 * 8, 16):
        p = ctypes.c_void_p()
        h = ctypes.create_string_buffer(64)
        _lib.check(L.tba_ipc_alloc(nbytes, ctypes.byref(p), h), "alloc")
        bufs.append(p.value)
    slots = torch.tensor([bufs[0], bufs[0]], dtype=torch.int64, device="cuda")   # "rank 1" never writes
    flags = torch.tensor([bufs[1], bufs[1] + 8], dtype=torch.int64, device="cuda")
    w = dataclasses.replace(syn.WORKLOADS["toy"])
    inp = H.device_inputs(w, 0)
    x = tba.make_rows(inp["logits"], inp["tokens"], inp["mask"])
    o = tba.ops._Fwd(w.N, w.K, torch.device("cuda"))
    ws = torch.empty(tba.workspace_bytes(w.N, w.T), dtype=torch.uint8, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    pr = TbaPeerReduce(slots.data_ptr(), flags.data_ptr(), 0, 2, 1, 0.2)
    rc = L.tba_tb_loss_fwd_peer(ctypes.byref(x), None, inp["ref_logp"].data_ptr(), inp["log_reward"].data_ptr(),
                                w.beta, w.K, float(w.N), ws.data_ptr(), o.seq_logp.data_ptr(), o.n_tokens.data_ptr(),
                                o.log_z.data_ptr(), o.resid.data_ptr(), o.partial.data_ptr(), ctypes.byref(pr),
                                st.data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    torch.cuda.synchronize()
    assert st.item() & _lib.TBA_DEV_PEER_TIMEOUT
    assert torch.isnan(o.partial).all()
    for p in bufs:
        L.tba_ipc_free(p)
