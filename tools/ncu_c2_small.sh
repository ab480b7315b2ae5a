#!/bin/bash
# ncu --set full of every small kernel of the c2 BbST_CON (bitmap) solve
out=gpurun_out/ncu_c2small; mkdir -p $out
N="ncu --set full --clock-control none --import-source on -c 1"
for k in k_collect k_piece_count k_block_argmin_keys_ml k_st_tile k_query_flat; do
  $N -k regex:$k -s 2 -o $out/$k -f python tools/prof.py --config c2 --variant con_bitmap --iters 3 > $out/$k.log 2>&1
done
echo done
