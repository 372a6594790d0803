python tools/attn_microbench.py --live 724 --trace
python tools/attn_microbench.py --live 724 --jitter 0 --trace
python tools/attn_microbench.py --live 2000 --trace
python tools/attn_microbench.py --live 724 --ctas 74
python tools/attn_microbench.py --live 724 --batch 1 --trace
