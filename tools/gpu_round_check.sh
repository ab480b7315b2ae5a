#!/bin/bash
# Round-end style check on the GPU box: -m gpu tests, smoke, bench (ours + the
# reference arm), the c2 launch list and one full ncu capture of the contraction.
tag=${1:-r02}
out=gpurun_out/$tag; mkdir -p $out
python -m pytest tests -m gpu -x -q > $out/gputests.log 2>&1; echo "rc=$?" >> $out/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "rc=$?" >> $out/smoke.log
python bench.py > $out/bench.json 2> $out/bench.err
python bench.py --impl reference --steps 5 --warmup 1 > $out/bench_ref.json 2> $out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_c2.csv \
    python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu > $out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_contract -s 1 -c 1 -o $out/contract_c2 -f \
    python tools/prof.py --iters 2 --variant con_bitmap > $out/ncu_contract.log 2>&1
echo done
