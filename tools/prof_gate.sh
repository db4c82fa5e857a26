# ncu evidence for the decode gate variants (cluster vs split-K fused) at T = 1 / 64
mkdir -p gpurun_out/pg
B="python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu --no-train --no-shapes"
python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "golden or q30_decode or shared or identity or k_equals or zero_init or fully_masked or determ" > gpurun_out/pg/tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/pg/tests.log
$B --tokens 1 > gpurun_out/pg/plain.log 2>&1 || exit 1
python tools/decode_points.py --T 1,8,64 --s 0,0.5,0.875 > gpurun_out/pg/points_cluster.jsonl 2>&1
for t in 1 64; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/pg/launches_T${t}_cluster.csv $B --tokens $t > /dev/null 2>&1; echo l$t=$?
done
ncu --set full --clock-control none --import-source on -k regex:gate_cluster -s 3 -c 1 -o gpurun_out/pg/gate_cluster_T1 $B --tokens 1 > gpurun_out/pg/ncu1.log 2>&1; echo n1=$?
ncu --set full --clock-control none --import-source on -k regex:gate_cluster -s 3 -c 1 -o gpurun_out/pg/gate_cluster_T64 $B --tokens 64 > gpurun_out/pg/ncu64.log 2>&1; echo n64=$?
