out=gpurun_out/ck2; mkdir -p $out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q > $out/gputests.log 2>&1; echo rc=$? >> $out/gputests.log; tail -2 $out/gputests.log
timeout 600 python tools/quick.py --configs c2,c3,c4,c5 --variants con_bitmap --check > $out/quick.log 2>&1; tail -4 $out/quick.log | cut -c1-220
BRMQ_LIB=ab/stamps.so timeout 300 python tools/contract_tail.py | head -5
