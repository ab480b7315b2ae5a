out=gpurun_out/q3; mkdir -p $out
export PYTHONUNBUFFERED=1
timeout 600 python tools/quick.py --configs c3,c4,c5 --variants bbst --check > $out/quick.log 2>&1
tail -3 $out/quick.log
timeout 900 python -m pytest tests -m gpu -x -q > $out/gputests.log 2>&1; echo rc=$? >> $out/gputests.log; tail -2 $out/gputests.log
