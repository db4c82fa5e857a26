for m in auto fused split; do
  BEAM_GATE_MODE=$m python tools/decode_points.py --T 1,8,64 --s 0,0.5,0.875 --steps 30
done
BEAM_GATE_MODE=fused python tools/gate_trace.py
