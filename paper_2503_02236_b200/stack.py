"""Graph-captured execution of a stack of fused VQ GEMVs (a decode step's linears).

``VQLinearStack`` is the public API a serving loop (and bench.py's end-to-end
leg) calls: it owns the quantized weights, device input/output buffers and one
CUDA graph that replays every GEMV of the stack, so a decode step costs one
graph launch instead of one Python->C-ABI round trip per layer.
"""

import torch

from . import _native as N
from .device import DeviceVQTensor, dtype_enum
from .ops import Workspace, launch_struct


class VQLinearStack:
    def __init__(self, weights, rows: int = 1, act_dtype=torch.float16, out_dtype=torch.float16,
                 launches=None, grouped: bool = False):
        self.weights = list(weights)
        if not self.weights:
            raise ValueError("empty stack")
        self.device = self.weights[0].device
        self.rows = rows
        self.act_dtype, self.out_dtype = act_dtype, out_dtype
        self.launches = list(launches) if launches else [launch_struct() for _ in self.weights]
        ins = [w.shape[0] for w in self.weights]
        outs = [w.shape[1] for w in self.weights]
        self.in_off = [0]
        for m in ins:
            self.in_off.append(self.in_off[-1] + rows * m)
        self.out_off = [0]
        for n in outs:
            self.out_off.append(self.out_off[-1] + rows * n)
        self.x = torch.zeros(self.in_off[-1], dtype=act_dtype, device=self.device)
        self.y = torch.zeros(self.out_off[-1], dtype=out_dtype, device=self.device)
        self._structs = [w.struct() for w in self.weights]
        lib = N.lib()
        need = max(N.check(lib.vqb_workspace_bytes(N.KERNEL_GEMV, s, rows, L))
                   for s, L in zip(self._structs, self.launches))
        # private arena: the graph bakes its pointer in (never the shared per-stream one)
        self._ws = Workspace(self.device, need).buf
        self._graph = None
        # grouped: the stack's (independent) GEMVs run as persistent launches of up to
        # GROUP_MAX problems each (vqb_gemv_grouped) instead of one launch per linear
        self.grouped = bool(grouped)
        self._groups = []
        if self.grouped:
            import ctypes
            esz_x, esz_y = self.x.element_size(), self.y.element_size()
            for g0 in range(0, len(self.weights), self.GROUP_MAX):
                idx = list(range(g0, min(g0 + self.GROUP_MAX, len(self.weights))))
                structs = (N.VqbTensor * len(idx))(*[self._structs[i] for i in idx])
                xs = (ctypes.c_void_p * len(idx))(*[self.x.data_ptr() + self.in_off[i] * esz_x for i in idx])
                ys = (ctypes.c_void_p * len(idx))(*[self.y.data_ptr() + self.out_off[i] * esz_y for i in idx])
                self._groups.append((structs, xs, ys, len(idx), self.launches[g0]))

    GROUP_MAX = 192

    @property
    def n_launches(self) -> int:
        return len(self._groups) if self.grouped else len(self.weights)

    def input_view(self, i: int) -> torch.Tensor:
        return self.x[self.in_off[i]:self.in_off[i + 1]].view(self.rows, -1)

    def output_view(self, i: int) -> torch.Tensor:
        return self.y[self.out_off[i]:self.out_off[i + 1]].view(self.rows, -1)

    def launch_all(self) -> None:
        """Enqueue every GEMV on the current stream (no host sync)."""
        lib = N.lib()
        stream = torch.cuda.current_stream(self.device).cuda_stream
        xd, yd = dtype_enum(self.act_dtype), dtype_enum(self.out_dtype)
        esz_x, esz_y = self.x.element_size(), self.y.element_size()
        xb, yb = self.x.data_ptr(), self.y.data_ptr()
        ws, wsn = self._ws.data_ptr(), self._ws.numel()
        if self.grouped:
            import ctypes
            for structs, xs, ys, n, L in self._groups:
                N.check(lib.vqb_gemv_grouped(ctypes.cast(structs, ctypes.c_void_p), n, ctypes.cast(xs, ctypes.c_void_p),
                                             xd, self.rows, ctypes.cast(ys, ctypes.c_void_p), yd, L, ws, wsn, stream))
            return
        for i, (s, L) in enumerate(zip(self._structs, self.launches)):
            N.check(lib.vqb_gemv(s, xb + self.in_off[i] * esz_x, xd, self.rows,
                                 yb + self.out_off[i] * esz_y, yd, L, ws, wsn, stream))

    def capture(self) -> None:
        """Record launch_all() into a CUDA graph (after one eager warm-up)."""
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            self.launch_all()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                self.launch_all()
        torch.cuda.current_stream(self.device).wait_stream(s)
        self._graph = g

    def replay(self) -> None:
        if self._graph is None:
            self.capture()
        self._graph.replay()

    def run(self, host_x: torch.Tensor, host_y: torch.Tensor) -> None:
        """End to end: pinned host inputs -> GPU stack -> pinned host outputs."""
        self.x.copy_(host_x, non_blocking=True)
        self.replay()
        host_y.copy_(self.y, non_blocking=True)


class StackPipeline:
    """Serving-loop form of ``VQLinearStack.run``: two device buffer sets (each with its
    own captured graph, sharing the weights) and separate host->device and
    device->host copy streams, so step k's input copy and step k-1's result copy overlap
    the neighbouring steps' compute. Every step still moves its inputs host->device and
    its result device->host; only the waiting is hidden (PCIe is full duplex)."""

    def __init__(self, stack: VQLinearStack):
        twin = VQLinearStack(stack.weights, rows=stack.rows, act_dtype=stack.act_dtype, out_dtype=stack.out_dtype,
                             launches=stack.launches, grouped=stack.grouped)
        self.sets = [stack, twin]
        for s in self.sets:
            if s._graph is None:
                s.capture()
        dev = stack.device
        self.h2d = torch.cuda.Stream(dev)
        self.d2h = torch.cuda.Stream(dev)
        self.in_ready = [torch.cuda.Event() for _ in range(2)]
        self.out_ready = [torch.cuda.Event() for _ in range(2)]
        self.set_free = [torch.cuda.Event() for _ in range(2)]

    def run(self, host_xs, host_ys) -> None:
        """One step per (pinned host input, pinned host output) pair, in order."""
        comp = torch.cuda.current_stream(self.sets[0].device)
        for k, (hx, hy) in enumerate(zip(host_xs, host_ys)):
            i = k % 2
            st = self.sets[i]
            with torch.cuda.stream(self.h2d):
                if k >= 2:
                    self.h2d.wait_event(self.set_free[i])  # this set's previous result is read out
                st.x.copy_(hx, non_blocking=True)
                self.in_ready[i].record(self.h2d)
            comp.wait_event(self.in_ready[i])
            st.replay()
            self.out_ready[i].record(comp)
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(self.out_ready[i])
                hy.copy_(st.y, non_blocking=True)
                self.set_free[i].record(self.d2h)
        comp.wait_stream(self.d2h)
        comp.wait_stream(self.h2d)
