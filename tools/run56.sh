for P in "" "--no-plan"; do
timeout 120 python tools/attn_microbench.py --live 724 $P; timeout 120 python tools/attn_microbench.py --live 724 --isolated $P
timeout 120 python tools/attn_microbench.py --live 724 --trace $P | head -1
done
