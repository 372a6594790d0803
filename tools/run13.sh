./tools/bulk_bw.bin
