# sparsity sweep + MMA-rate microbenchmark (run under gpurun; 1 GPU).  Writes gpurun_out/.
set -x
python -c "import __graft_entry__ as g; g.build()"
./bench_micro/mma_rate > gpurun_out/mma_rate.log 2>&1; cat gpurun_out/mma_rate.log
timeout 1200 python scripts/sweep.py --out gpurun_out/r01_sweep.jsonl > gpurun_out/sweep.log 2>&1; tail -5 gpurun_out/sweep.log
