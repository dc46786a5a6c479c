#!/bin/bash
# Evidence for the end of round 2 (the shipped library: drain votes per 64 columns, fused seed set-up, per-thread workspaces): ncu launch list + full
# captures, probe tests, config table, sweeps, sanitizer logs.  Output: gpurun_out/*_r2c.*
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU="ncu --clock-control none"
timeout 900 $NCU --metrics gpu__time_duration.sum -c 800 --csv --log-file gpurun_out/launches_r2c_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extras > gpurun_out/ncu_bench_r2c.log 2>&1; echo "launch list rc=$?"
timeout 900 $NCU --set full --import-source on -k regex:scan_queue_kernel -s 1 -c 1 -f -o gpurun_out/prof_queue_r2c python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-extras > gpurun_out/ncu_full_r2c.log 2>&1; echo "full queue rc=$?"
ncu -i gpurun_out/prof_queue_r2c.ncu-rep --page raw --csv > gpurun_out/ncu_full_umma_queue_r2c.csv 2>/dev/null
ncu -i gpurun_out/prof_queue_r2c.ncu-rep --page source --csv > gpurun_out/src_queue_r2c.csv 2>/dev/null && python tools/ncu_hot.py gpurun_out/src_queue_r2c.csv 30 > gpurun_out/ncu_hot_umma_queue_r2c.txt 2>&1
timeout 300 python tools/umma_profile.py 10000 > gpurun_out/umma_profile_r2c.log 2>&1
bash tools/bench_configs.sh > gpurun_out/configs_r2c.jsonl 2>&1; echo "configs rc=$?"
python tools/batch_sweep.py 10000000 256 100 > gpurun_out/sweep_10m_256_r2c.jsonl 2>&1
python tools/batch_sweep.py 1000000 768 100 1,16,64,1024,10000 > gpurun_out/sweep_1m_768_r2c.jsonl 2>&1
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --num-cuda-barriers 4096 python tools/umma_one.py seeded > gpurun_out/${t}_umma_seeded_r2c.log 2>&1; echo "$t umma rc=$?"
done
timeout 600 python tools/queue_stress.py > gpurun_out/queue_stress_r2c.log 2>&1; echo "queue stress rc=$?"
timeout 900 python tools/umma_stress.py 1 60 > gpurun_out/umma_stress_r2c.log 2>&1; echo "stress rc=$?"
rm -f gpurun_out/*.ncu-rep gpurun_out/src_*.csv
for f in gpurun_out/memcheck_*_r2c.log gpurun_out/racecheck_*_r2c.log gpurun_out/synccheck_*_r2c.log; do
  if [ -f "$f" ] && [ $(stat -c %s "$f") -gt 200000 ]; then (head -150 "$f"; echo "[... $(wc -l < "$f") lines in all ...]"; grep -E "SUMMARY|match|k_select|small batch" "$f" | tail -12) > "$f.tmp" && mv "$f.tmp" "$f"; fi
done
ls -la gpurun_out | grep r2c
