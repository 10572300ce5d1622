#!/bin/bash
# One GPU-box pass: bench line, ncu launch list of the same bench command,
# and a full ncu capture of one pipeline run (per-kernel traffic, stalls),
# summarised on the box (the .ncu-rep stays there unless KEEP_REP=1).
# Usage (under gpurun): bash tools/gpu_profile.sh [config] [extra bench args]
cfg=${1:-2}
shift
mkdir -p gpurun_out
if [ "${SKIP_BENCH:-0}" != 1 ]; then
python bench.py --config "$cfg" --no-extra-configs "$@" > gpurun_out/bench_c$cfg.json 2> gpurun_out/bench_c$cfg.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/launches_c$cfg.csv \
    python bench.py --config "$cfg" --steps 2 --warmup 3 --no-cpu-baseline --no-extra-configs > gpurun_out/ncu_launch_c$cfg.log 2>&1
fi
rep=/tmp/full_c$cfg
ncu --set full --metrics lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum --clock-control none --import-source on -k 'regex:^k_|DeviceScan' -c ${NCU_COUNT:-60} \
    -o $rep -f python tools/tune.py --config "$cfg" --reps 1 > gpurun_out/ncu_full_c$cfg.log 2>&1
python tools/ncu_sum.py $rep.ncu-rep > gpurun_out/ncu_sum_c$cfg.txt 2>&1
python tools/ncu_traffic.py $rep.ncu-rep $cfg > gpurun_out/ncu_traffic_c$cfg.log 2>&1
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
for k in k_w_gather k_edge_search k_edge_fix k_out_lists k_link_tour k_link_rows k_walk k_positions k_propose k_compress k_tile k_chunk_rows k_heads; do
  python tools/ncu_lines.py $rep.ncu-rep $k 0 12
done > gpurun_out/ncu_lines_c$cfg.txt 2>&1
if [ "${KEEP_REP:-0}" = 1 ]; then cp $rep.ncu-rep gpurun_out/; fi
echo done
