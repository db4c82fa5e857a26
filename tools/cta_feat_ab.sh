for rep in 1 2; do for f in 4 8; do
  BEAM_CTA_FEAT=$f python tools/decode_points.py --T 1,2 --s 0,0.5,0.875 --steps 60 | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); print('feat=$f', r['T'], r['s'], r['us'], r['stages_eager_us']['experts_gateup'])"
done; done
