"""Eager batch-1 decode steps for an ncu launch list (per-kernel durations of one step).
Usage: ncu --metrics gpu__time_duration.sum --csv ... python tools/decode_kernel_times.py [batch]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_02236_b200.decode import LlamaShape, VQLlamaDecoder  # noqa: E402

b = int(sys.argv[1]) if len(sys.argv) > 1 else 1
dev = torch.device("cuda", 0)
dec = VQLlamaDecoder.synthetic(LlamaShape(), b, 4096, dev)
dec.set_length(4000)
for _ in range(3):
    dec.run_step()
torch.cuda.synchronize()
