mkdir -p gpurun_out
for lib in base cur; do
  if [ $lib = base ]; then export BEAM_LIB=$PWD/tools/ab_base.so; else unset BEAM_LIB; fi
  for s in 0 0.875; do
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"gateup|down_|gate_fused|combine" --csv --log-file gpurun_out/k_${lib}_$s.csv python tools/decode_points.py --T 1 --s $s --steps 3 > /dev/null 2>&1
    python tools/ncu_kernels.py gpurun_out/k_${lib}_$s.csv "$lib s=$s"
  done
done
