REPS=1 ncu --set full --clock-control none --import-source on -k regex:"k_forward" -c 1 -o gpurun_out/prof_span python tools/one_view.py > gpurun_out/ncu_span.log 2>&1
