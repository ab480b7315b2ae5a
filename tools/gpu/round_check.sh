# GPU tests + bench (no sweep) into gpurun_out/$1
out=gpurun_out/${1:-chk}; mkdir -p $out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q > $out/gputests.log 2>&1; echo rc=$? >> $out/gputests.log
timeout 600 python bench.py --no-sweep > $out/bench.json 2> $out/bench.err
tail -3 $out/gputests.log
python - "$out" <<'P'
import json, sys
d = json.loads(open(sys.argv[1] + '/bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['preprocess'], d['stages_ms'], d['variants_queries_per_s'], d['bit_exact_vs_reference'])
for k, v in d.get('configs', {}).items(): print(k, v)
P
