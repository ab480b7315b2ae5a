out=gpurun_out/nc1; mkdir -p $out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_contract -s 1 -c 1 -o $out/contract_c2 -f python tools/prof.py --iters 2 --variant con_bitmap > $out/ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_query_flat -s 1 -c 1 -o $out/query_c2 -f python tools/prof.py --iters 2 --variant con_bitmap > $out/ncu_q.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_piece_count -s 1 -c 1 -o $out/piece_c2 -f python tools/prof.py --iters 2 --variant con_bitmap > $out/ncu_p.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_collect -s 1 -c 1 -o $out/collect_c2 -f python tools/prof.py --iters 2 --variant con_bitmap > $out/ncu_c.log 2>&1
ls -la $out
