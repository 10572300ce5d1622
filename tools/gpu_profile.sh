#!/bin/bash
# One GPU-box pass: bench line, ncu launch list of the same bench command,
# and a full ncu capture of one pipeline run (per-kernel traffic, stalls).
# Usage (under gpurun): bash tools/gpu_profile.sh [config] [extra bench args]
cfg=${1:-2}
shift
mkdir -p gpurun_out
python bench.py --config "$cfg" "$@" > gpurun_out/bench_c$cfg.json 2> gpurun_out/bench_c$cfg.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/launches_c$cfg.csv \
    python bench.py --config "$cfg" --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_c$cfg.log 2>&1
ncu --set full --clock-control none --import-source on -k 'regex:^k_|DeviceScan' -c 60 \
    -o gpurun_out/full_c$cfg -f python tools/tune.py --config "$cfg" --reps 1 > gpurun_out/ncu_full_c$cfg.log 2>&1
echo done
