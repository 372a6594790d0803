for L in 309 724 2000; do timeout 120 python tools/attn_microbench.py --live $L; timeout 120 python tools/attn_microbench.py --live $L --isolated; done
