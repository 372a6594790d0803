nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2507_16784_b200/csrc tools/bulk_bw.cu -o /tmp/bulk_bw && /tmp/bulk_bw
