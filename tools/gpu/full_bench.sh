# full bench (sweep + configs) + reference arm + c2 launch list
out=gpurun_out/${1:-fb}; mkdir -p $out
export PYTHONUNBUFFERED=1
timeout 1200 python bench.py > $out/bench.json 2> $out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $out/bench_ref.json 2> $out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu > $out/ncu_launch.log 2>&1
python tools/ncu_summary.py launches $out/launches_c2.csv > $out/launches_c2_summary.txt 2>&1
tail -1 $out/bench.json | cut -c1-300; tail -1 $out/bench_ref.json | cut -c1-300
