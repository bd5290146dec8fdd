#!/bin/bash
# The round's measurement set on one B200 (run under gpurun from the repo root): bench lines
# (config 3 default, config 2, deterministic, reference arm), the ncu launch list of the bench
# command and one --set full capture of a fused config-3 view.  Outputs in gpurun_out/prof/.
set -u
O=gpurun_out/prof
mkdir -p $O
timeout 400 python bench.py > $O/bench.json 2> $O/bench.err
timeout 400 python bench.py --resolution 64 --image 512 --views 4 > $O/bench_config2.json 2> $O/bench_config2.err
timeout 400 python bench.py --deterministic > $O/bench_deterministic.json 2> $O/bench_det.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference_arm.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 > $O/ncu_launch.log 2>&1
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_forward|k_backward|k_cull_emit|k_window_counts|k_tile_sort|k_chain|k_bin" -o $O/full \
  python tools/one_view_fused.py > $O/ncu_full.log 2>&1
ls -la $O
