mkdir -p gpurun_out/prof
B="python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu --no-train --no-shapes"
python tools/e2e_probe.py > gpurun_out/prof/e2e_probe.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/prof/launches_T1.csv $B --tokens 1 > /dev/null 2>&1; echo l1=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/prof/launches_T64.csv $B --tokens 64 > /dev/null 2>&1; echo l64=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/prof/launches_T8192.csv $B --tokens 8192 --sparsity 0 > /dev/null 2>&1; echo l8k=$?
ncu --set full --clock-control none --import-source on -k regex:gateup_ffma -s 4 -c 1 -o gpurun_out/prof/gateup_T64 $B --tokens 64 > gpurun_out/prof/ncu_gateup.log 2>&1; echo f1=$?
ncu --set full --clock-control none --import-source on -k regex:grouped_gemm_2sm -s 4 -c 2 -o gpurun_out/prof/gemm_T8192 $B --tokens 8192 --sparsity 0 > gpurun_out/prof/ncu_gemm.log 2>&1; echo f2=$?
ncu --set full --clock-control none --import-source on -k regex:gate_fused -s 4 -c 1 -o gpurun_out/prof/gate_T64 $B --tokens 64 > gpurun_out/prof/ncu_gate.log 2>&1; echo f3=$?
ncu --set full --clock-control none --import-source on -k regex:_mma_kernel -s 8 -c 2 -o gpurun_out/prof/mma_T64_s0 $B --tokens 64 --sparsity 0 > gpurun_out/prof/ncu_mma.log 2>&1; echo f4=$?
