timeout 120 python tools/gpu/repro3.py 300000/40000 1000003/100000 70001/5000 1000003/7 2>&1 | tail -1
timeout 300 python tools/quick.py --configs c1,c2,c3,c4,c5 --variants con_bitmap,con_radix --check | cut -c1-150
for i in 1 2; do timeout 300 python tools/quick.py --configs c2 --variants con_bitmap --steps 30 | cut -c1-110; BRMQ_PIECE_COUNT=1 timeout 300 python tools/quick.py --configs c2 --variants con_bitmap --steps 30 | cut -c1-110; done
timeout 500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
