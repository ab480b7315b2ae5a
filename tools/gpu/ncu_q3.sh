out=gpurun_out/nq3; mkdir -p $out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_query -s 1 -c 1 -o $out/query_c3 -f python tools/prof.py --config c3 --variant bbst --iters 2 > $out/ncu.log 2>&1
tail -2 $out/ncu.log
