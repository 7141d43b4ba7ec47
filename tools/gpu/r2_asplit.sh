for s in 1 2 3 4 6 8 12 16; do timeout 120 python tools/attn_bench.py --p 560 --split $s; done
