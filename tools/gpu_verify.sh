set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --no-cpu --precision bf16 > gpurun_out/bench_bf16.json 2>&1
timeout 600 python bench.py --no-cpu --config c3 > gpurun_out/bench_c3.json 2>&1
timeout 600 python bench.py --no-cpu --config c5 > gpurun_out/bench_c5.json 2>&1
tail -3 gpurun_out/pytest_gpu.log
tail -1 gpurun_out/bench_c2.json
