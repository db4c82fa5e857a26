# Per-kernel ncu durations of tools/ab_base.so (base) vs the in-tree library (cur)
# on one decode_points workload.  usage: bash tools/ncu_ab.sh <T> "<s list>" "<kernel regex>"
T=${1:-1}; SS=${2:-"0 0.875"}; KRE=${3:-"gateup|down_|gate_fused|combine"}
mkdir -p gpurun_out
for lib in base cur; do
  if [ $lib = base ]; then export BEAM_LIB=$PWD/tools/ab_base.so; else unset BEAM_LIB; fi
  for s in $SS; do
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"$KRE" --csv \
      --log-file gpurun_out/k_${lib}_$s.csv python tools/decode_points.py --T $T --s $s --steps 3 > /dev/null 2>&1
    python tools/ncu_kernels.py gpurun_out/k_${lib}_$s.csv "$lib s=$s"
  done
done
