mkdir -p gpurun_out/r02b
python tools/decode_points.py --T 1,8,16,32,64 --s 0,0.5,0.875 --steps 30 > gpurun_out/r02b/points.jsonl 2>&1
cat gpurun_out/r02b/points.jsonl | python -c "
import sys,json
for l in sys.stdin:
    try: r=json.loads(l)
    except Exception: print(l.strip()); continue
    print(r['T'], r['s'], r['us'], r['stages_eager_us'])"
B="python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu --no-train --no-shapes"
ncu --set full --clock-control none --import-source on -k regex:grouped_gemm -s 4 -c 2 -o /tmp/gemm_T8192 $B --tokens 8192 --sparsity 0 > gpurun_out/r02b/gemm.log 2>&1; echo gemm=$?
python tools/ncu_export.py /tmp/gemm_T8192.ncu-rep "T=8192 s=0" gpurun_out/r02b > gpurun_out/r02b/export.log 2>&1
ncu -i /tmp/gemm_T8192.ncu-rep --page raw --csv > gpurun_out/r02b/gemm_raw.csv 2>/dev/null
cp profiles/ncu_summary.json gpurun_out/r02b/
