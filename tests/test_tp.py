"""Tensor-parallel sharding + collectives on CPU (gloo, world size 2).

Local compute is the CPU oracle here (test infrastructure); on GPUs the same
TPLinear / TPAttention run the CUDA kernels and NCCL.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp
from conftest import Case, O
from paper_2503_02236_b200.device import stack_codebooks


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _dense(q):
    regs = O.region_ids(q.shape, q.config.vector_size, q.config.sharing.kind,
                        (q.config.sharing.tile_rows, q.config.sharing.tile_cols), q.config.sharing.group_width)
    return O.dequantize(q.codes, stack_codebooks(q), q.shape, q.config.vector_size, q.n_regions, regs)


def _oracle_linear(w, x):
    return torch.from_numpy(O.matmul_ref(x.numpy(), _dense(w)))


def _oracle_attention(k, v, q):
    return torch.from_numpy(O.attention_ref(q.numpy(), _dense(k), _dense(v)))


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2503_02236_b200.tp import TPAttention, TPLinear
    try:
        out = {}
        for name in ("gptvq2", "quip2", "aqlm2x8", "cg2d"):
            q = Case(name).quantized()
            x = torch.from_numpy(O.synthetic_tensor((3, q.shape[0]), 5))
            full = O.matmul_ref(x.numpy(), _dense(q))
            col = TPLinear.from_full(q, "column", compute=_oracle_linear)(x).numpy()
            out[f"col_{name}"] = O.rel_err(col, full)
            if name != "cg2d":
                row = TPLinear.from_full(q, "row", compute=_oracle_linear)(x).numpy()
                out[f"row_{name}"] = O.rel_err(row, full)
        k, v = Case("cq4").quantized(), Case("cq4", seed_offset=1).quantized()
        b, h, t, c = k.shape
        qv = torch.from_numpy(O.synthetic_tensor((b, h, c), 9))
        full = O.attention_ref(qv.numpy(), _dense(k), _dense(v))
        att = TPAttention.from_full(k, v, compute=_oracle_attention)(qv).numpy()
        out["attn_cq4"] = O.rel_err(att, full)
        if rank == 0:
            results.update(out)
    finally:
        dist.destroy_process_group()


def test_tensor_parallel_gloo_world2():
    port = _free_port()
    with mp.Manager() as mgr:
        results = mgr.dict()
        mp.spawn(_worker, args=(2, port, results), nprocs=2, join=True)
        res = dict(results)
    assert res, "rank 0 reported nothing"
    for key, err in res.items():
        assert err <= 1e-5, (key, err)


def test_shard_validation():
    from paper_2503_02236_b200.errors import ConfigError, ShapeError
    from paper_2503_02236_b200.tp import shard_columns, shard_heads
    q = Case("gptvq2").quantized()        # 512 columns, 256-column tiles
    with pytest.raises(ConfigError):
        shard_columns(q, 0, 4)            # 128-column shards would split a codebook tile
    with pytest.raises(ShapeError):
        shard_columns(q, 0, 3)
    k = Case("cq4").quantized()
    s = shard_heads(k, 1, 2)
    assert s.shape == (2, 2, 64, 128) and s.n_regions == 2 * 64
    # the shard's books are the second half of the heads' books
    np.testing.assert_array_equal(s.codebook_for(0, 0).entries, k.codebook_for(0, 2 * 64).entries)
