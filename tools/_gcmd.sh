python tools/phases.py > gpurun_out/phases.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>gpurun_out/bench.err
python bench.py --no-cpu-baseline > gpurun_out/bench2.log 2>>gpurun_out/bench.err
