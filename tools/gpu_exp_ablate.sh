for s in "" front silu norm attn linear; do echo "skip=$s $(VQB_DECODE_SKIP=$s python tools/decode_bench.py 1 --reps 20)"; done
