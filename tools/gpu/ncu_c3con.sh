out=gpurun_out/nc3c; mkdir -p $out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_contract -s 1 -c 1 -o $out/contract_c3con -f python tools/prof.py --config c3 --iters 2 --variant con_bitmap > $out/ncu.log 2>&1
tail -1 $out/ncu.log
