# A/B of the grouped-GEMM producer's TMA L2 prefetch distance (BEAM_GEMM_PREFETCH_KB)
for pf in 0 4 8 16; do
  BEAM_GEMM_PREFETCH_KB=$pf python tools/decode_points.py --T 8192 --s 0,0.5,0.85 --steps 5 | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); print('pf=$pf', r['T'], r['s'], r['us'])"
done
