# A/B of two library builds on the same box: tools/ab_base.so (a previous commit)
# vs the current in-tree library, interleaved.  usage: bash tools/lib_ab.sh "<decode_points args>"
ARGS=${1:-"--T 1,2 --s 0,0.5,0.875 --steps 60"}
for rep in 1 2; do
  for lib in base cur; do
    if [ $lib = base ]; then export BEAM_LIB=$PWD/tools/ab_base.so; else unset BEAM_LIB; fi
    python tools/decode_points.py $ARGS | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); print('$lib', r['T'], r['s'], r['us'])"
  done
done
