"""End-to-end Llama decode with VQ weights and a CQ-quantized KV cache.

The reference stops at single fused kernels; this module chains them into the decode
step the paper evaluates end to end: per layer

    RMSNorm(+residual) -> fused VQ GEMV qkv -> RoPE -> online CQ quantization of the
    new K/V rows (reference quantize, codec.py:367-389) -> decode attention over the
    CQ cache -> VQ GEMV o -> RMSNorm(+residual) -> VQ GEMV gate|up -> SiLU*up ->
    VQ GEMV down

then the final RMSNorm, a dense fp16 LM head (cuBLAS, a plain library GEMM) and the
next-token draw (`vqb_sample`: greedy, or temperature / top-k by Gumbel-max). The current length lives in a device int32 that the step advances
itself, so one CUDA graph replays every decode step while the cache grows.
Batches of up to 64 rows take the decode GEMV (CUDA cores, mma.sync or tcgen05 by batch
size), larger batches the tcgen05 GEMM.
"""

import os
from dataclasses import dataclass

import torch

from .codec import Sharing, VQConfig
from . import _native as N
from . import ops
from .device import DeviceVQTensor
from .errors import CapacityError, ConfigError


@dataclass(frozen=True)
class LlamaShape:
    hidden: int = 4096
    heads: int = 32
    head_dim: int = 128
    ffn: int = 11008
    layers: int = 32
    vocab: int = 32000
    rope_theta: float = 10000.0
    eps: float = 1e-5


WEIGHT_CFG = VQConfig(8, 16, 1)  # QuiP#-style E8 VQ (BASELINE C2)
KV_CFG = VQConfig(2, 8, 1, Sharing.per_channel_group(2))  # CQ-4 (BASELINE C4)


@dataclass
class DecoderLayer:
    qkv: DeviceVQTensor      # (hidden, 3*hidden): [q | k | v]
    o: DeviceVQTensor        # (hidden, hidden)
    gate_up: DeviceVQTensor  # (hidden, 2*ffn): [gate | up]
    down: DeviceVQTensor     # (ffn, hidden)
    attn_norm: torch.Tensor
    ffn_norm: torch.Tensor
    k_cache: DeviceVQTensor  # (B, heads, T_cap, head_dim) CQ codes
    v_cache: DeviceVQTensor


class VQLlamaDecoder:
    def __init__(self, shape: LlamaShape, layers, embed: torch.Tensor, final_norm: torch.Tensor,
                 lm_head: torch.Tensor, batch: int, group=None, tp_world: int = 1):
        self.shape = shape
        self.layers = list(layers)
        self.embed = embed          # (vocab, hidden) fp16
        self.final_norm = final_norm
        self.lm_head = lm_head      # (hidden, vocab) fp16: logits = x @ lm_head
        self.batch = batch
        self.device = embed.device
        # tensor parallelism (Megatron): this rank holds heads [h0, h1) of qkv / the KV
        # caches and its slice of ffn; o and down are row-parallel and all-reduced
        self.group = group           # None = the default process group when tp_world > 1
        self.world = int(tp_world)
        self.comm = None             # tp.PeerComm: row-parallel all-reduce fused into the GEMV (peer memory)
        self.local_heads = self.layers[0].k_cache.shape[1] if self.layers else shape.heads
        self.d_len = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.tokens = torch.zeros(batch, dtype=torch.int64, device=self.device)
        self.res = torch.zeros((batch, shape.hidden), dtype=torch.float16, device=self.device)
        self.res_b = torch.zeros_like(self.res)  # ping-pong partner for the norm fused into the GEMV
        self.logits = None
        self._graph = None
        self.length = 0  # host mirror of d_len (the step advances both)
        self.ws = ops.Workspace(self.device)  # private arena the captured graph keeps alive
        # next-token rule (vqb_sample): greedy by default; set_sampling before capture()
        self.temperature, self.top_k, self.seed, self.top_p = 0.0, 0, 0, 1.0
        self.capacity = min(L.k_cache.shape[2] for L in self.layers) if self.layers else 0
        # batch 1: the fused gate_up projection is stored interleaved per 128 columns,
        # [gate 128 | up 128] in every 256-column block, so its GEMV epilogue emits
        # silu(gate) * up directly (VQB_XF_SWIGLU_OUT) — one kernel less per layer
        f_local = self.layers[0].gate_up.shape[1] // 2 if self.layers else 0
        self.gu_il = (batch == 1 and self.layers and f_local % 128 == 0
                      and all(L.gate_up.layout == "gemv" for L in self.layers))
        if self.gu_il:
            for L in self.layers:
                L.gate_up = self._interleave_gate_up(L.gate_up)

    # -- construction -------------------------------------------------------------------------

    @staticmethod
    def _interleave_gate_up(w: DeviceVQTensor) -> DeviceVQTensor:
        """[gate | up] (F + F columns) -> [gate 128 | up 128] per 256-column block."""
        from .tp import device_shard
        f = w.shape[1] // 2
        ranges = []
        for c0 in range(0, f, 128):
            ranges += [(c0, c0 + 128), (f + c0, f + c0 + 128)]
        return device_shard(w, col_ranges=ranges)

    @staticmethod
    def _gate_up_ranges(f: int, lo: int, hi: int, interleaved: bool):
        """Column ranges of gate[lo:hi] then up[lo:hi] in a gate_up weight stored
        [gate | up] or interleaved per 128 columns."""
        if not interleaved:
            return [(lo, hi), (f + lo, f + hi)]
        gate, up = [], []
        c = lo
        while c < hi:
            blk, off = divmod(c, 128)
            n = min(hi - c, 128 - off)
            gate.append((blk * 256 + off, blk * 256 + off + n))
            up.append((blk * 256 + 128 + off, blk * 256 + 128 + off + n))
            c += n
        return gate + up

    def _silu(self, gu: torch.Tensor) -> torch.Tensor:
        """silu(gate) * up of a gate_up output in this decoder's column layout."""
        if self.gu_il:
            b, n = gu.shape
            gu = gu.view(b, n // 256, 2, 128).permute(0, 2, 1, 3).reshape(b, n).contiguous()
        return ops.silu_mul(gu)

    @staticmethod
    def synthetic(shape: LlamaShape, batch: int, capacity: int, device, seed: int = 0, working_entries: int = 256):
        """Random weights of the named architecture (no checkpoints offline): codes
        from the working set, N(0, 0.1) books; CQ books per head and channel group."""
        g = torch.Generator(device=device)
        g.manual_seed(seed)
        d, f = shape.hidden, shape.ffn

        def vq_weight(m, n):
            s = m * n // WEIGHT_CFG.vector_size
            codes = torch.randint(0, working_entries, (1, s), generator=g, device=device, dtype=torch.int32)
            books = (torch.randn((1, WEIGHT_CFG.n_entries, WEIGHT_CFG.vector_size), generator=g, device=device)
                     * (0.5 / m ** 0.5)).half()
            return DeviceVQTensor.from_device_codes(codes, (m, n), WEIGHT_CFG, books).relayout("gemv")

        def kv_cache():
            groups = shape.head_dim // KV_CFG.vector_size
            books = torch.randn((shape.heads * groups, 256, KV_CFG.vector_size), generator=g, device=device).half()
            return DeviceVQTensor.empty_cache((batch, shape.heads, capacity, shape.head_dim), KV_CFG, books)

        layers = []
        for _ in range(shape.layers):
            layers.append(DecoderLayer(
                vq_weight(d, 3 * d), vq_weight(d, d), vq_weight(d, 2 * f), vq_weight(f, d),
                torch.ones(d, dtype=torch.float16, device=device), torch.ones(d, dtype=torch.float16, device=device),
                kv_cache(), kv_cache()))
        embed = torch.randn((shape.vocab, d), generator=g, device=device).half()
        lm_head = (torch.randn((d, shape.vocab), generator=g, device=device) / d ** 0.5).half()
        return VQLlamaDecoder(shape, layers, embed, torch.ones(d, dtype=torch.float16, device=device), lm_head, batch)

    # -- the step -----------------------------------------------------------------------------

    gemv_max_rows = 64  # batches up to this take the decode GEMV (CUDA cores 1-3, mma.sync 4, tcgen05 5-64)
    fuse_norms = True  # batch 1: RMSNorm / SiLU gating fused into the following GEMV's prologue
    fuse_append = True  # RoPE + KV append inside the attention kernel (CQ-4 caches at C = 128)
    fuse_append_max_batch = 8  # measured: the separate append kernel wins from batch 16

    def _attend(self, L: DecoderLayer, qkv: torch.Tensor) -> torch.Tensor:
        """RoPE, online KV quantization of the new token and decode attention: one fused
        launch when the caches allow it, else qkv_rope_append + vq_attention."""
        sh = self.shape
        # measured: fused wins at batch 1-8 (1.83 vs 1.88 ms at 1, 3.07 vs 3.19 at 4); from 16
        # rows the CTA holding each (b, h)'s last chunk serialises too many quantizations
        if (self.fuse_append and self.batch <= self.fuse_append_max_batch and L.k_cache.shape[3] == 128 and L.k_cache.config == KV_CFG
                and L.k_cache.layout == "kv"):
            return ops.vq_attention_append(L.k_cache, L.v_cache, qkv, self.d_len, sh.rope_theta)
        q = ops.qkv_rope_append(qkv, L.k_cache, L.v_cache, self.d_len, sh.rope_theta)
        return ops.vq_attention(L.k_cache, L.v_cache, q, out_dtype=torch.float16, d_len=self.d_len)

    def _linear(self, w: DeviceVQTensor, x: torch.Tensor) -> torch.Tensor:
        if x.shape[0] <= self.gemv_max_rows:
            return ops.vq_gemv(w, x, out_dtype=torch.float16)
        return ops.vq_gemm(w, x, out_dtype=torch.float16)

    def _reduce(self, y: torch.Tensor) -> torch.Tensor:
        """Sum a row-parallel linear's partial output over the TP group."""
        if self.world > 1:
            torch.distributed.all_reduce(y, group=self.group)
        return y

    def _row_linear(self, w: DeviceVQTensor, x: torch.Tensor) -> torch.Tensor:
        """A row-parallel linear and its all-reduce: fused over peer memory when the
        decoder holds a PeerComm and the batch takes the GEMV, else GEMV/GEMM + NCCL."""
        if self.comm is not None and x.shape[0] in (1, 2, 4, 8, 16):
            return self.comm.linear(w, x, "row", out_dtype=torch.float16)
        return self._reduce(self._linear(w, x))

    @classmethod
    def tensor_parallel(cls, full: "VQLlamaDecoder", group, rank: int = None, world: int = None,
                        fused_collectives: bool = False) -> "VQLlamaDecoder":
        """This rank's shard of a decoder (same weights): qkv columns of heads
        [h0, h1) for q, k and v, o rows of those heads, gate/up columns of ffn slice
        [f0, f1), down rows of it, KV caches (and their per-head CQ books) of the
        local heads. Embedding, norms and LM head are replicated."""
        from .tp import device_shard
        if world is None:
            world, rank = torch.distributed.get_world_size(group), torch.distributed.get_rank(group)
        sh = full.shape
        if sh.heads % world or sh.ffn % world:
            raise ConfigError(f"heads {sh.heads} / ffn {sh.ffn} not divisible by tensor-parallel size {world}")
        hl, fl, c, d = sh.heads // world, sh.ffn // world, sh.head_dim, sh.hidden
        h0, f0 = rank * hl, rank * fl
        hcols = [(part * d + h0 * c, part * d + (h0 + hl) * c) for part in range(3)]
        layers = []
        for L in full.layers:
            groups = c // KV_CFG.vector_size

            def cache(src):
                books = src.codebooks[h0 * groups:(h0 + hl) * groups].contiguous()
                return DeviceVQTensor.empty_cache((full.batch, hl, src.shape[2], c), KV_CFG, books)

            layers.append(DecoderLayer(
                device_shard(L.qkv, col_ranges=hcols), device_shard(L.o, rows=(h0 * c, (h0 + hl) * c)),
                device_shard(L.gate_up, col_ranges=cls._gate_up_ranges(sh.ffn, f0, f0 + fl, full.gu_il)),
                device_shard(L.down, rows=(f0, f0 + fl)), L.attn_norm, L.ffn_norm, cache(L.k_cache),
                cache(L.v_cache)))
        # the collectives run only in a real process group (rank / world given without
        # one emulate a shard, e.g. to check it in a single process)
        live = torch.distributed.is_initialized()
        dec = cls(sh, layers, full.embed, full.final_norm, full.lm_head, full.batch, group=group,
                  tp_world=world if live else 1)
        if fused_collectives and live and world > 1:
            from .tp import PeerComm
            dec.comm = PeerComm(full.batch, sh.hidden, group=group, device=full.device)
        return dec

    def step(self) -> torch.Tensor:
        """One decode step for the current tokens; returns (and stores) the next ones.
        Device-side only (capturable): the length counter advances first, so every
        kernel of the step sees the new token's position as d_len - 1.

        VQB_DECODE_SKIP (comma list of norm, linear, front, attn, silu) drops stages
        for time attribution only — the output is then meaningless."""
        with ops.use_workspace(self.ws):
            return self._step()

    def _step(self) -> torch.Tensor:
        skip = set(filter(None, os.environ.get("VQB_DECODE_SKIP", "").split(",")))
        if skip:
            return self._step_ablated(skip)
        sh, b = self.shape, self.batch
        ops.add_len(self.d_len, 1)
        self.res.copy_(torch.index_select(self.embed, 0, self.tokens))
        x = None
        hc = self.local_heads * sh.head_dim
        if self.fuse_norms and b == 1 and self.gemv_max_rows >= 1:
            return self._step_fused()
        for L in self.layers:
            xn = ops.rmsnorm(x, self.res, L.attn_norm, sh.eps)
            qkv = self._linear(L.qkv, xn)
            a = self._attend(L, qkv)
            o = self._row_linear(L.o, a.view(b, hc))
            xn = ops.rmsnorm(o, self.res, L.ffn_norm, sh.eps)
            gu = self._linear(L.gate_up, xn)
            x = self._row_linear(L.down, self._silu(gu))
        xn = ops.rmsnorm(x, self.res, self.final_norm, sh.eps)
        self.logits = xn @ self.lm_head
        return self._sample()

    def _step_fused(self) -> torch.Tensor:
        """Batch-1 step with the norms and the SiLU gate fused into the GEMVs that
        consume them (vqb_gemv_xf): per layer qkv(+attn norm), rope/append, attention,
        o, gate_up(+ffn norm), down(+SiLU) — 6 launches instead of 9. The residual
        stream alternates between two buffers (every CTA of a fused GEMV reads the old
        one while CTA 0 writes the new one); same arithmetic as the unfused step."""
        sh = self.shape
        res = (self.res, self.res_b)
        cur = 0
        x = None
        hc = self.local_heads * sh.head_dim
        for L in self.layers:
            qkv = ops.vq_gemv_rmsnorm(L.qkv, x, res[cur], L.attn_norm, sh.eps, residual_out=res[1 - cur])
            cur ^= 1
            a = self._attend(L, qkv)
            o = self._row_linear(L.o, a.view(1, hc))
            if self.gu_il:
                # ffn norm in the prologue, SiLU gating in the epilogue of the gate_up GEMV
                h = ops.vq_gemv_rmsnorm(L.gate_up, o, res[cur], L.ffn_norm, sh.eps, residual_out=res[1 - cur],
                                        swiglu=True)
            else:
                h = self._silu(ops.vq_gemv_rmsnorm(L.gate_up, o, res[cur], L.ffn_norm, sh.eps,
                                                   residual_out=res[1 - cur]))
            cur ^= 1
            x = self._row_linear(L.down, h)
        xn = ops.rmsnorm(x, res[cur], self.final_norm, sh.eps)
        self.logits = xn @ self.lm_head
        return self._sample()

    def _step_ablated(self, skip):
        sh, b = self.shape, self.batch
        ops.add_len(self.d_len, 1)
        self.res.copy_(torch.index_select(self.embed, 0, self.tokens))
        hc = sh.heads * sh.head_dim
        xn = torch.zeros((b, sh.hidden), dtype=torch.float16, device=self.device)
        qkv = torch.zeros((b, 3 * hc), dtype=torch.float16, device=self.device)
        q = torch.zeros((b, sh.heads, sh.head_dim), dtype=torch.float16, device=self.device)
        a = torch.zeros((b, sh.heads, sh.head_dim), dtype=torch.float16, device=self.device)
        gu = torch.zeros((b, 2 * sh.ffn), dtype=torch.float16, device=self.device)
        hm = torch.zeros((b, sh.ffn), dtype=torch.float16, device=self.device)
        x = None
        for L in self.layers:
            if "norm" not in skip:
                xn = ops.rmsnorm(x, self.res, L.attn_norm, sh.eps)
            if "linear" not in skip:
                qkv = self._linear(L.qkv, xn)
            if "front" not in skip:
                q = ops.qkv_rope_append(qkv, L.k_cache, L.v_cache, self.d_len, sh.rope_theta)
            if "attn" not in skip:
                a = ops.vq_attention(L.k_cache, L.v_cache, q, out_dtype=torch.float16, d_len=self.d_len)
            o = self._linear(L.o, a.view(b, hc)) if "linear" not in skip else xn
            if "norm" not in skip:
                xn = ops.rmsnorm(o, self.res, L.ffn_norm, sh.eps)
            if "linear" not in skip:
                gu = self._linear(L.gate_up, xn)
            if "silu" not in skip:
                hm = self._silu(gu)
            x = self._linear(L.down, hm) if "linear" not in skip else xn
        xn = ops.rmsnorm(x, self.res, self.final_norm, sh.eps)
        self.logits = xn @ self.lm_head
        return self._sample()

    def set_sampling(self, temperature: float = 0.0, top_k: int = 0, seed: int = 0, top_p: float = 1.0) -> None:
        """Temperature / top-k / top-p sampling of the next token (Gumbel-max over the logits,
        noise hashed from the seed and the device length, so every replayed step draws
        afresh and TP ranks draw identically). temperature 0 = greedy. A captured graph
        keeps the rule it was captured with: call this before capture()."""
        if temperature < 0 or top_k < 0 or not 0 < top_p <= 1:
            raise ConfigError("sampling needs temperature >= 0, top_k >= 0 and 0 < top_p <= 1")
        self.temperature, self.top_k, self.seed, self.top_p = float(temperature), int(top_k), int(seed), float(top_p)

    def _sample(self) -> torch.Tensor:
        return ops.sample(self.logits, self.temperature, self.top_k, self.seed, d_step=self.d_len, out=self.tokens,
                          top_p=self.top_p)

    def capture(self) -> None:
        """Record one step as a CUDA graph. The warm-up step (on the capture stream)
        and the capture itself advance the length and the tokens, so both are restored;
        the KV rows they wrote sit at the position the first replay overwrites."""
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        saved_len, saved_tok = self.d_len.clone(), self.tokens.clone()
        with torch.cuda.stream(s), ops.use_workspace(self.ws):
            self.step()
            self.d_len.copy_(saved_len)
            self.tokens.copy_(saved_tok)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                self.step()
            self.d_len.copy_(saved_len)
            self.tokens.copy_(saved_tok)
        torch.cuda.current_stream(self.device).wait_stream(s)
        self._graph = g

    def _advance(self) -> None:
        """A step writes the new token's K/V rows at position `length`: refuse
        to step past the cache capacity (the kernels would skip the write and flag
        the device error word)."""
        if self.length + 1 > self.capacity:
            raise CapacityError(f"KV cache full: {self.length} tokens cached, capacity {self.capacity}")
        self.length += 1

    def replay(self) -> None:
        if self._graph is None:
            self.capture()
        self._advance()
        self._graph.replay()

    def run_step(self) -> torch.Tensor:
        """One eager (uncaptured) step with the capacity check."""
        self._advance()
        return self.step()

    def set_length(self, n: int) -> None:
        """Pretend n tokens are already cached (benchmarks at a fixed context)."""
        n = int(n)
        if n < 0 or n >= self.capacity:
            raise CapacityError(f"length {n} outside [0, {self.capacity}) of the KV cache")
        self.d_len.fill_(n)
        self.length = n

    def check_device_errors(self) -> None:
        """Raise if any KV append since the last check fell outside the cache."""
        if N.take_device_error() & 1:
            raise CapacityError("a KV append position fell outside the cache capacity (write skipped)")
