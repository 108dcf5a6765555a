#!/bin/bash
# Round-2 profiling pass on one B200 (run under gpurun from the repo root).
# Launch lists are cold-cache serialised replays: compare shares, not absolutes.
set -u
O=gpurun_out/r02
mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
# graph-replayed decode times over gamma, fixed 30 and early stop
python tools/kbench.py --graph --decode-only --gammas 32 64 128 256 512 1024 2048 4096 --reps 20 > $O/kbench_graph.jsonl 2>&1
python tools/kbench.py --graph --decode-only --early-stop --gammas 1024 4096 --reps 12 >> $O/kbench_graph.jsonl 2>&1
# per-kernel device times of a gamma-32 decode (graph off: one launch per kernel)
ncu --metrics $M --clock-control none --csv --log-file $O/launches_g32.csv \
    python tools/kbench.py --decode-only --gammas 32 --reps 1 > /dev/null 2>&1
# LDPCCC slot kernels, 18360' I=20 gamma 512 and I=5 gamma 128
python tools/sbench.py --gamma 512 --I 20 --steps 2 > $O/sbench.jsonl 2>&1
python tools/sbench.py --gamma 128 --I 5 --steps 4 >> $O/sbench.jsonl 2>&1
python tools/sbench.py --gamma 512 --I 5 --steps 4 >> $O/sbench.jsonl 2>&1
ncu --metrics $M --clock-control none -s 1200 -c 400 --csv --log-file $O/launches_stream_I20_g512.csv \
    python tools/sbench.py --gamma 512 --I 20 --steps 1 --no-graph > /dev/null 2>&1
ncu --metrics $M --clock-control none -s 400 -c 400 --csv --log-file $O/launches_stream_I5_g128.csv \
    python tools/sbench.py --gamma 128 --I 5 --steps 2 --no-graph > /dev/null 2>&1
# full captures: LDPCCC check pass, fused block kernel
ncu --set full --clock-control none --import-source on -k regex:check_kernel -s 300 -c 1 -o $O/prof_scheck \
    python tools/sbench.py --gamma 512 --I 20 --steps 1 --no-graph > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:agg_fused -s 10 -c 1 -o $O/prof_fused \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --stream-gamma 0 --sustain-s 0 --no-curve > /dev/null 2>&1
ncu --metrics $M --clock-control none -k regex:agg_fused -s 10 -c 20 --csv --log-file $O/traffic_fused_g1024.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --stream-gamma 0 --sustain-s 0 --no-curve > /dev/null 2>&1
ls -la $O
