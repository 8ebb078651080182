# GPU check (run under gpurun): parity tests, smoke, a short bench.  Writes gpurun_out/.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -30 > gpurun_out/pytest_attn.log
cat gpurun_out/pytest_attn.log
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
cat gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -5 gpurun_out/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; tail -5 gpurun_out/bench.log
