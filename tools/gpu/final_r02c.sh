# round-2c evidence: full bench (sweep + configs) + reference arm + c2 launch list,
# then ncu --set full of the c2 contraction and query and the c5-con MSD marking
tag=${1:-r02c}
bash tools/gpu/full_bench.sh fb_$tag
out=gpurun_out/ncu_$tag; mkdir -p $out
N="timeout 600 ncu --set full --clock-control none --import-source on -c 1 -f"
$N -k regex:k_contract -s 1 -o $out/contract_c2 python tools/prof.py --iters 2 --variant con_bitmap > $out/contract_c2.log 2>&1
$N -k regex:k_query_flat -s 1 -o $out/query_c2 python tools/prof.py --iters 2 --variant con_bitmap > $out/query_c2.log 2>&1
$N -k regex:k_msd_partition -s 1 -o $out/partition_c5con python tools/prof.py --config c5 --variant con_bitmap --iters 2 > $out/partition_c5con.log 2>&1
$N -k regex:k_bucket_mark -s 1 -o $out/bucket_c5con python tools/prof.py --config c5 --variant con_bitmap --iters 2 > $out/bucket_c5con.log 2>&1
ls -la $out
