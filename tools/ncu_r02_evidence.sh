#!/bin/bash
# One ncu --set full capture per kernel named in VERDICT r01 "evidence gaps"
# (run on the GPU box: gpurun -- bash tools/ncu_r02_evidence.sh <tag>).
tag=${1:-r02}
out=gpurun_out/ncu_$tag
mkdir -p $out
N="ncu --set full --clock-control none --import-source on -c 1"
$N -k regex:k_block_argmin_i32_vec -s 1 -o $out/k1_c3 -f python tools/prof.py --config c3 --variant bbst --iters 2 > $out/k1_c3.log 2>&1
$N -k regex:k_block_argmin_i32_vec -s 1 -o $out/k1_c5 -f python tools/prof.py --config c5 --variant bbst --iters 2 > $out/k1_c5.log 2>&1
$N -k regex:k_st_tile -s 3 -o $out/k2_c5 -f python tools/prof.py --config c5 --variant bbst --iters 2 > $out/k2_c5.log 2>&1
$N -k regex:k_collect -s 1 -o $out/collect_c5con -f python tools/prof.py --config c5 --variant con_bitmap --iters 2 > $out/collect_c5con.log 2>&1
$N -k regex:k_rs_pass -s 4 -o $out/rs_pass_c5con -f python tools/prof.py --config c5 --variant con_radix --iters 2 > $out/rs_pass_c5con.log 2>&1
$N -k regex:k_query -s 1 -o $out/query_c3 -f python tools/prof.py --config c3 --variant bbst --iters 2 > $out/query_c3.log 2>&1
echo done
