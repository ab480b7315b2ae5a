# full-chain PDL (BRMQ_PDL=1) against the default (contraction + query only)
BRMQ_PDL=1 timeout 300 python tools/quick.py --configs c1,c2,c3,c4,c5 --variants con_bitmap,con_radix,bbst --check | cut -c1-110
for i in 1 2 3; do for p in 0 1; do
  echo -n "PDL=$p "; BRMQ_PDL=$p timeout 300 python tools/quick.py --configs c1,c2 --variants con_bitmap --steps 40 | cut -c1-70 | tr '\n' ' '; echo
done; done
for p in 0 1; do echo -n "PDL=$p "; BRMQ_PDL=$p timeout 300 python tools/quick.py --configs c3,c5 --variants con_bitmap,bbst --steps 10 | cut -c1-70 | tr '\n' ' '; echo; done
