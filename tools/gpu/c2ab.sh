timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --cache-control none -k regex:k_contract -c 8 --csv --log-file gpurun_out/c2ab.csv python tools/quick.py --configs c2 --variants con_bitmap --steps 3 > /dev/null 2>&1
grep -o '"smsp__inst_executed.sum","inst","[0-9,.]*"\|"gpu__time_duration.sum","ns","[0-9,.]*"' gpurun_out/c2ab.csv | tail -4
for i in 1 2; do timeout 300 python tools/quick.py --configs c2 --variants con_bitmap --steps 30 | cut -c1-140; done
timeout 300 python tools/quick.py --configs c1,c3,c4,c5 --variants con_bitmap,con_radix --check | cut -c1-150
