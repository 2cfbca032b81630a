"""Fused tensor-parallel collectives over peer memory (csrc/tp.cu, tp.PeerComm;
SURVEY.md §8f row 4) with two processes on the test box's one B200: the symmetric
buffers are mapped across the processes with CUDA IPC, the GEMV epilogue pushes
its outputs into both ranks' slots and the finish kernel reduces / gathers them.

* TPLinear row (all-reduce) and column (all-gather) with the fused collective
  against the oracle on the full tensors, repeated so the epochs cycle through
  both slot parities;
* the Megatron-sharded Llama decoder with fused all-reduces after o and down
  matches the single-process decoder's logits, eagerly and replayed as a CUDA graph;
* no rank ever timed out waiting for its peer (error word 0).
"""

import os

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _init_file():
    # file rendezvous: no TCP port to race for between tests (a freed port can be
    # taken again before the workers bind it)
    import tempfile
    return os.path.join(tempfile.mkdtemp(prefix="vqb_tp_"), "rendezvous")


def _worker(rank, world, init_file, results):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for p in (root, os.path.join(root, "tests"), os.path.join(root, "tests", "golden")):
        if p not in sys.path:
            sys.path.insert(0, p)
    import torch
    import torch.distributed as dist
    from conftest import Case, O
    dist.init_process_group("gloo", init_method=f"file://{init_file}", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    from paper_2503_02236_b200 import _native as N
    from paper_2503_02236_b200.decode import LlamaShape, VQLlamaDecoder
    from paper_2503_02236_b200.device import stack_codebooks
    from paper_2503_02236_b200.tp import PeerComm, TPLinear
    out = {}
    try:
        def dense(q):
            sh = q.config.sharing
            regs = O.region_ids(q.shape, q.config.vector_size, sh.kind, (sh.tile_rows, sh.tile_cols), sh.group_width)
            return O.dequantize(q.codes, stack_codebooks(q), q.shape, q.config.vector_size, q.n_regions, regs)

        comm = PeerComm(max_rows=8, max_n=4096, device=dev)
        for name in ("quip2", "aqlm2x8"):
            q = Case(name, books_f16=True).quantized()
            for mode in ("row", "column"):
                lin = TPLinear.from_full(q, mode, device=dev)
                lin.comm = comm
                for it, rows in enumerate((1, 2, 8)):
                    x = O.round_f16(O.synthetic_tensor((rows, q.shape[0]), 5 + it))
                    full = O.matmul_ref(x, dense(q))
                    y = lin(torch.from_numpy(x).to(dev).half())
                    kern = N.last_kernel()
                    out[f"{mode}_{name}_b{rows}"] = (O.rel_err(y.float().cpu().numpy(), full), kern)
        out["linear_timeouts"] = (float(comm.take_error()), "tp_finish")
        comm.close()

        sh = LlamaShape(hidden=512, heads=4, head_dim=128, ffn=1024, layers=2, vocab=256)
        full_dec = VQLlamaDecoder.synthetic(sh, 2, 64, dev, seed=5)
        tp_dec = VQLlamaDecoder.tensor_parallel(full_dec, None, fused_collectives=True)
        assert tp_dec.comm is not None
        toks = torch.tensor([3, 11], device=dev)
        full_dec.tokens.copy_(toks)
        tp_dec.tokens.copy_(toks)
        errs = []
        for _ in range(3):
            full_dec.run_step()
            tp_dec.run_step()
            errs.append(O.rel_err(tp_dec.logits.float().cpu().numpy(), full_dec.logits.float().cpu().numpy()))
        tp_dec.capture()
        for _ in range(3):
            full_dec.run_step()
            tp_dec.replay()
            errs.append(O.rel_err(tp_dec.logits.float().cpu().numpy(), full_dec.logits.float().cpu().numpy()))
        out["decoder_logits"] = (max(errs), "decode")
        out["decoder_timeouts"] = (float(tp_dec.comm.take_error()), "tp_finish")
        tp_dec.comm.close()
        if rank == 0:
            results.update(out)
    finally:
        dist.destroy_process_group()


def test_fused_peer_memory_collectives_world2():
    import torch.multiprocessing as mp
    init_file = _init_file()
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        results = mgr.dict()
        mp.spawn(_worker, args=(2, init_file, results), nprocs=2, join=True)
        res = dict(results)
    assert res, "rank 0 reported nothing"
    for key, (err, kern) in res.items():
        if key.endswith("timeouts"):
            assert err == 0, key
            continue
        tol = 3e-2 if key == "decoder_logits" else 2e-3
        assert err <= tol, (key, err, kern)
        if key != "decoder_logits":
            assert kern == "tp_finish", (key, kern)
