out=gpurun_out/nqf; mkdir -p $out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_query_flat -s 1 -c 1 -o $out/qflat_c3con -f python tools/prof.py --config c3 --variant con_bitmap --iters 2 > $out/ncu.log 2>&1
tail -1 $out/ncu.log
