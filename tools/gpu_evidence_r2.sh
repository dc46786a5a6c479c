#!/bin/bash
# Round-2 evidence in one GPU session: ncu launch list + full captures, sanitizer logs, config table.  Output: gpurun_out/
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NCU="ncu --clock-control none"
timeout 900 $NCU --metrics gpu__time_duration.sum -c 800 --csv --log-file gpurun_out/launches_r2_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extras > gpurun_out/ncu_bench_r2.log 2>&1; echo "launch list rc=$?"
timeout 900 $NCU --set full --import-source on -k regex:scan_queue_kernel -s 1 -c 1 -f -o gpurun_out/prof_queue_r2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-extras > gpurun_out/ncu_full_r2.log 2>&1; echo "full queue rc=$?"
ncu -i gpurun_out/prof_queue_r2.ncu-rep --page raw --csv > gpurun_out/ncu_full_umma_queue_r2.csv 2>/dev/null
ncu -i gpurun_out/prof_queue_r2.ncu-rep --page source --csv > gpurun_out/src_queue_r2.csv 2>/dev/null && python tools/ncu_hot.py gpurun_out/src_queue_r2.csv 30 > gpurun_out/ncu_hot_umma_queue_r2.txt 2>&1
timeout 900 $NCU --set full --import-source on -k regex:search_kernel -s 4 -c 1 -f -o gpurun_out/prof_coop_r2 python tools/batch_sweep.py 10000000 256 100 4 > gpurun_out/ncu_coop_r2.log 2>&1; echo "full coop rc=$?"
ncu -i gpurun_out/prof_coop_r2.ncu-rep --page raw --csv > gpurun_out/ncu_full_coop_search_r2.csv 2>/dev/null
ncu -i gpurun_out/prof_coop_r2.ncu-rep --page source --csv > gpurun_out/src_coop_r2.csv 2>/dev/null && python tools/ncu_hot.py gpurun_out/src_coop_r2.csv 30 > gpurun_out/ncu_hot_coop_search_r2.txt 2>&1
timeout 900 $NCU --set full -k regex:scan_queue_kernel -s 4 -c 1 -f -o gpurun_out/prof_q256_r2 python tools/batch_sweep.py 10000000 256 100 256 > gpurun_out/ncu_q256_r2.log 2>&1; echo "full nq256 rc=$?"
ncu -i gpurun_out/prof_q256_r2.ncu-rep --page raw --csv > gpurun_out/ncu_full_umma_queue_nq256_r2.csv 2>/dev/null
timeout 600 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches_r2_nq1.csv python tools/batch_sweep.py 10000000 256 100 1 > /dev/null 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches_r2_nq256.csv python tools/batch_sweep.py 10000000 256 100 256 > /dev/null 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum -k regex:hist_kernel --csv --log-file gpurun_out/launches_r2_estimate_scale.csv python - > gpurun_out/estimate_scale_r2.log 2>&1 <<'PY'
import sys, time; sys.path.insert(0, ".")
import torch, bench, paper_2008_02002_b200 as xb
x = bench.gen_rows_gpu(torch, 0, 4_000_000, 4_000_000, 256)
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter(); s = xb.estimate_scale(x, 0.98); torch.cuda.synchronize()
    print("estimate_scale 4M x 256 float32 on device:", round((time.perf_counter() - t0) * 1e3, 2), "ms, scale", s)
PY
bash tools/bench_configs.sh > gpurun_out/configs_r2.jsonl 2>&1; echo "configs rc=$?"
python tools/batch_sweep.py 1000000 768 100 1,16,64,1024,10000 > gpurun_out/sweep_1m_768_r2.jsonl 2>&1
python tools/batch_sweep.py 10000000 256 100 > gpurun_out/sweep_10m_256_r2.jsonl 2>&1
python tools/kselect_latency.py 10000000 0 > gpurun_out/kselect_r2.log 2>&1; python tools/kselect_latency.py 2000000 1 >> gpurun_out/kselect_r2.log 2>&1
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --num-cuda-barriers 4096 python tools/umma_one.py seeded > gpurun_out/${t}_umma_seeded_r2.log 2>&1; echo "$t umma rc=$?"
  timeout 900 compute-sanitizer --tool $t python tools/coop_one.py > gpurun_out/${t}_coop_r2.log 2>&1; echo "$t coop rc=$?"
done
for v in 0 1 4 5; do compute-sanitizer --tool racecheck tools/bin/sanitizer_probe $v 2>&1 | grep -E "variant|RACECHECK SUMMARY"; done > gpurun_out/racecheck_probe_r2.log 2>&1
for v in 2 3; do compute-sanitizer --tool synccheck tools/bin/sanitizer_probe $v 2>&1 | grep -E "variant|ERROR SUMMARY|Barrier error" | sort | uniq -c; done > gpurun_out/synccheck_probe_r2.log 2>&1
timeout 900 python tools/umma_stress.py 1 60 > gpurun_out/umma_stress_r2.log 2>&1; echo "stress rc=$?"
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_r2.log
rm -f gpurun_out/*.ncu-rep gpurun_out/src_*.csv   # only the exported summaries travel back (64 MiB limit)
for f in gpurun_out/memcheck_*_r2.log gpurun_out/racecheck_*_r2.log gpurun_out/synccheck_*_r2.log; do   # keep heads + summaries of the sanitizer logs
  if [ -f "$f" ] && [ $(stat -c %s "$f") -gt 200000 ]; then (head -150 "$f"; echo "[... $(wc -l < "$f") lines in all ...]"; grep -E "SUMMARY|match|k_select|small batch" "$f" | tail -12) > "$f.tmp" && mv "$f.tmp" "$f"; fi
done
du -sh gpurun_out; ls -la gpurun_out | tail -45
