out=gpurun_out/pc; mkdir -p $out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 60 --csv --log-file $out/l.csv python tools/quick.py --configs c2 --variants con_bitmap --steps 5 > /dev/null 2>&1
python tools/ncu_summary.py launches $out/l.csv | grep -v "at::"
for i in 1 2; do timeout 300 python tools/quick.py --configs c2 --variants con_bitmap --steps 30 | cut -c1-100; done
