# LPT tail assignment check (run under gpurun; 1 GPU): attention parity with the new default,
# interleaved timing of SV_TAIL_LPT=0/1 builds, a short bench
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/pytest_tail.log; cat gpurun_out/pytest_tail.log
SV_ROUNDS=15 timeout 600 python scripts/time_variants.py variants/lib_tail0.so variants/lib_tail1.so > gpurun_out/tail_variants.log 2>&1; tail -20 gpurun_out/tail_variants.log
SV_BH=16 SV_ROUNDS=15 timeout 600 python scripts/time_variants.py variants/lib_tail0.so variants/lib_tail1.so > gpurun_out/tail_variants16.log 2>&1; tail -20 gpurun_out/tail_variants16.log
timeout 600 python bench.py > gpurun_out/bench_tail.log 2>&1; tail -1 gpurun_out/bench_tail.log
