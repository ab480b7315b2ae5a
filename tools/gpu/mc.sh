timeout 300 python tools/quick.py --configs c1,c2,c3,c4,c5 --variants con_bitmap --check | cut -c1-150
for i in 1 2; do timeout 300 python tools/quick.py --configs c2 --variants con_bitmap --steps 30 | cut -c1-110; BRMQ_MARK_COUNT=0 timeout 300 python tools/quick.py --configs c2 --variants con_bitmap --steps 30 | cut -c1-110; done
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
