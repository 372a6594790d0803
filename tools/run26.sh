nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2507_16784_b200/csrc tools/bulk_bw.cu -o /tmp/bulk_bw && /tmp/bulk_bw
for L in 309 724 2000; do timeout 120 python tools/attn_microbench.py --live $L --trace; done
timeout 120 python tools/attn_microbench.py --live 724 --batch 512 --trace
