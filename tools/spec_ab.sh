# A/B of the speculative L2 warm-up of gate/up weights (BEAM_SPEC_L2_MB)
for mb in 0 64 96; do
  BEAM_SPEC_L2_MB=$mb python tools/decode_points.py --T 16,32,64 --s 0,0.5,0.875 --steps 40 | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); print('spec_mb=$mb', r['T'], r['s'], r['E_act'], r['us'])"
done
