for C in "3.0,0.75" "4.0,1.2" "4.0,1.6" "6.0,2.0"; do
 echo "cost $C"
 for A in "" "--ext 12 --n 180" "--ext 3 --n 60" "--ext 1 --n 20"; do TIMRUN_EXT_COST=$C timeout 120 python tools/attn_mixed_bench.py --only mode2 $A | cut -c1-60; done
done
