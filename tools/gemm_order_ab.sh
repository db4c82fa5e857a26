# A/B of the grouped-GEMM unit order (BEAM_GEMM_ORDER: GEMM1 digit, GEMM2 digit)
for o in 00 01 10 11; do
  BEAM_GEMM_ORDER=$o python tools/decode_points.py --T 8192 --s 0,0.5,0.85 --steps 5 | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); print('order=$o', r['T'], r['s'], r['us'])"
done
