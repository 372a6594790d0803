timeout 120 python tools/attn_microbench.py --live 724 --trace --dump
