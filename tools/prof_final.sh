# Final round-2 ncu evidence: launch lists + one `--set full` capture of every repo
# kernel of one layer call at the headline / latency / prefill workloads.  The
# reports are exported to text on the box (tools/ncu_export.py) and deleted: the
# .ncu-rep files are too large to bring back.
mkdir -p gpurun_out/fin
B="python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu --no-train --no-shapes"
K='regex:gate_fused|router_gemv|topk_mask|permute|gateup|down_|combine|pack_x|grouped_gemm'
$B --tokens 64 > gpurun_out/fin/plain64.log 2>&1 || { echo plain-failed; exit 1; }
for spec in "64 0.5" "64 0" "1 0.875" "1 0" "8192 0"; do
  set -- $spec
  ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
      --log-file gpurun_out/fin/launches_T$1_s$2.csv $B --tokens $1 --sparsity $2 > /dev/null 2>&1; echo "launches T=$1 s=$2 rc=$?"
done
full() {  # tokens sparsity skip count
  ncu --set full --clock-control none --import-source on -k "$K" -s $3 -c $4 \
      -o /tmp/full_T$1_s$2 $B --tokens $1 --sparsity $2 > gpurun_out/fin/full_T$1_s$2.log 2>&1; echo "full T=$1 s=$2 rc=$?"
  python tools/ncu_export.py /tmp/full_T$1_s$2.ncu-rep "T=$1 s=$2" gpurun_out/fin >> gpurun_out/fin/export.log 2>&1
  rm -f /tmp/full_T$1_s$2.ncu-rep
}
full 64 0.5 12 6
full 64 0 12 6
full 1 0.875 8 5
full 8192 0 14 9
cp profiles/ncu_summary.json gpurun_out/fin/ncu_summary.json
