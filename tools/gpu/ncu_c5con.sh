out=gpurun_out/nc5c; mkdir -p $out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_contract -s 1 -c 1 -o $out/contract_c5con -f python tools/prof.py --config c5 --iters 2 --variant con_radix > $out/ncu.log 2>&1
tail -1 $out/ncu.log
