# A/B of the device-side MMA-vs-FFMA item thresholds (tokens per active expert)
for gu in 3 2 1; do for dn in 2 1; do
  BEAM_MMA_TOK_GU=$gu BEAM_MMA_TOK_DN=$dn python tools/decode_points.py --T 8,16,32,64 --s 0,0.5,0.875 --steps 30 | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); print('gu=$gu dn=$dn', r['T'], r['s'], r['E_act'], r['us'])"
done; done
