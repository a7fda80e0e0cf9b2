#!/usr/bin/env bash
# Regenerate the measured evidence under profiles/ on a B200 box, e.g.
#   gpurun --timeout 3000 -- 'bash tools/refresh_profiles.sh r2'
# then copy gpurun_out/<round>/ summaries into profiles/ (see the end).
# Each ncu capture runs only after the same command has exited 0 without ncu.
set -u
R=${1:-r2}
O=gpurun_out/$R
mkdir -p "$O"

timeout 1200 python -m pytest tests -m gpu -q > "$O/pytest_gpu.txt" 2>&1; tail -1 "$O/pytest_gpu.txt"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$O/smoke.txt" 2>&1; tail -1 "$O/smoke.txt"

# bench lines (BASELINE metric; cfg5 -- the sharded mixdown -- is the default workload)
timeout 900 python bench.py > "$O/bench_cfg5.json" 2> "$O/bench_cfg5.err" && echo "cfg5 ok"
timeout 900 python bench.py --impl reference > "$O/bench_reference.json" 2> "$O/bench_reference.err" && echo "reference ok"
timeout 900 python bench.py --workload cfg2 > "$O/bench_cfg2.json" 2> "$O/bench_cfg2.err" && echo "cfg2 ok"
timeout 900 python bench.py --workload cfg4 --steps 3 > "$O/bench_cfg4.json" 2> "$O/bench_cfg4.err" && echo "cfg4 ok"
timeout 900 python bench.py --workload cfg4 --impl reference --steps 3 --warmup 1 > "$O/bench_cfg4_reference.json" 2>&1 && echo "cfg4 ref ok"
timeout 900 python bench.py --workload cfg3 --steps 5 > "$O/bench_cfg3.json" 2> "$O/bench_cfg3.err" && echo "cfg3 ok"
timeout 900 python tools/sweep_cfg3.py --check > "$O/cfg3_sweep.jsonl" 2> /dev/null && echo "cfg3 sweep ok"
timeout 600 python tools/power_probe.py > "$O/power.txt" 2>&1 && echo "power ok"
for w in 8 4 2; do
  timeout 900 python tools/shard_cfg5.py --steps 20 --world $w > "$O/cfg5_shards_n$w.json" 2> /dev/null && echo "shards n$w ok"
done
timeout 600 python tools/mix_check.py --full > "$O/mix_check_full.txt" 2>&1 && echo "mix_check ok"

# ncu: launch lists (cold-cache, serialised) and one --set full capture of the dominant kernels
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 400 --csv \
  --log-file "$O/launches_cfg5.csv" python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-fused \
  > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 400 --csv \
  --log-file "$O/launches_cfg2.csv" python bench.py --workload cfg2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline \
  > /dev/null 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_mix_mma -s 2 -c 1 \
  -o "$O/mix_mma_full" -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-fused > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_render_mma -s 4 -c 2 \
  -o "$O/render_mma_full" -f python bench.py --workload cfg2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
  > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --clock-control none --csv \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --log-file "$O/cfg3_points.csv" python tools/cfg3_points_ncu.py run > "$O/cfg3_points.jsonl" 2> /dev/null
echo "ncu done"

# back in the container:
#   cp gpurun_out/$R/bench_*.json profiles/${R}_...   (and the other json/jsonl files)
#   python tools/ncu_summary.py --launches gpurun_out/$R/launches_cfg5.csv > profiles/${R}_cfg5_launches.txt
#   python tools/ncu_summary.py gpurun_out/$R/mix_mma_full.ncu-rep > profiles/${R}_cfg5_k_mix_mma_full.txt
#   python tools/ncu_summary.py gpurun_out/$R/render_mma_full.ncu-rep > profiles/${R}_cfg2_k_render_mma_full.txt
#   python tools/cfg3_points_ncu.py summarize gpurun_out/$R/cfg3_points.csv gpurun_out/$R/cfg3_points.jsonl > profiles/${R}_cfg3_points_ncu.txt
#   update profiles/traffic.json (dram bytes of one mix / one render launch) from those summaries
