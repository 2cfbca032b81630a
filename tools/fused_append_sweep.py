import sys, os, json, torch
sys.path.insert(0, os.getcwd())
from paper_2503_02236_b200.decode import LlamaShape, VQLlamaDecoder
dev = torch.device("cuda", 0)
for b in (1, 2, 4, 8):
    for fa in (True, False):
        dec = VQLlamaDecoder.synthetic(LlamaShape(), b, 4096, dev)
        dec.fuse_append = fa
        dec.set_length(4096 - 1 - 20 - 3)
        dec.capture()
        for _ in range(3): dec.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): dec.replay()
        e1.record(); torch.cuda.synchronize()
        print(b, fa, round(e0.elapsed_time(e1) / 20, 3), flush=True)
        del dec; torch.cuda.empty_cache()
