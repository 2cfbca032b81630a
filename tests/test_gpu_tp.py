"""Tensor parallelism with the CUDA kernels, two processes on the one
B200 of the test box: torch.distributed with the gloo backend moves the CUDA
tensors (NCCL refuses two ranks on one device); on an 8-GPU node the same code
runs one rank per GPU over NCCL.

* TPLinear column / row and TPAttention by head, local compute = the sm_100a
  kernels, against the oracle on the full tensors;
* the Llama decoder sharded Megatron-style (qkv / gate_up column-parallel, o / down
  row-parallel + all-reduce, KV cache by head) produces the single-process
  decoder's logits step after step.
"""

import os

import numpy as np
import pytest
from conftest import Case, O

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
    from paper_2503_02236_b200.tp import TPAttention, TPLinear
    out = {}
    try:
        def dense(q):
            sh = q.config.sharing
            regs = O.region_ids(q.shape, q.config.vector_size, sh.kind, (sh.tile_rows, sh.tile_cols), sh.group_width)
            return O.dequantize(q.codes, stack_codebooks(q), q.shape, q.config.vector_size, q.n_regions, regs)

        for name in ("quip2", "aqlm2x8", "gptvq2"):
            q = Case(name, books_f16=True).quantized()
            x = O.round_f16(O.synthetic_tensor((2, q.shape[0]), 5))
            full = O.matmul_ref(x, dense(q))
            xt = torch.from_numpy(x).to(dev).half()
            col = TPLinear.from_full(q, "column", device=dev)(xt).float().cpu().numpy()
            out[f"col_{name}"] = (O.rel_err(col, full), N.last_kernel())
            row = TPLinear.from_full(q, "row", device=dev)(xt).float().cpu().numpy()
            out[f"row_{name}"] = (O.rel_err(row, full), N.last_kernel())
        k, v = Case("cq4", books_f16=True).quantized(), Case("cq4", seed_offset=1, books_f16=True).quantized()
        b, h, t, c = k.shape
        qv = O.round_f16(O.synthetic_tensor((b, h, c), 9))
        full = O.attention_ref(qv, dense(k), dense(v))
        att = TPAttention.from_full(k, v, device=dev)(torch.from_numpy(qv).to(dev).half()).float().cpu().numpy()
        out["attn_cq4"] = (O.rel_err(att, full), N.last_kernel())

        sh = LlamaShape(hidden=512, heads=4, head_dim=128, ffn=1024, layers=2, vocab=256)
        full_dec = VQLlamaDecoder.synthetic(sh, 2, 64, dev, seed=5)
        tp_dec = VQLlamaDecoder.tensor_parallel(full_dec, None)
        assert tp_dec.local_heads == sh.heads // world
        toks = torch.tensor([3, 11], device=dev)
        full_dec.tokens.copy_(toks)
        tp_dec.tokens.copy_(toks)
        errs = []
        for _ in range(4):
            full_dec.run_step()
            tp_dec.run_step()
            errs.append(O.rel_err(tp_dec.logits.float().cpu().numpy(), full_dec.logits.float().cpu().numpy()))
        out["decoder_logits"] = (max(errs), "decode")
        if rank == 0:
            results.update(out)
    finally:
        dist.destroy_process_group()


def test_tensor_parallel_cuda_kernels_world2():
    import torch.multiprocessing as mp
    init_file = _init_file()
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        results = mgr.dict()
        mp.spawn(_worker, args=(2, init_file, results), nprocs=2, join=True)
        res = dict(results)
    assert res, "rank 0 reported nothing"
    for key, (err, kern) in res.items():
        tol = 3e-2 if key == "decoder_logits" else 2e-3
        assert err <= tol, (key, err, kern)
        if key != "decoder_logits":
            assert kern in ("gemv_fast", "gemv_generic", "attn_cq"), (key, kern)
