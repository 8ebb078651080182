# softmax-state-in-smem check (run under gpurun; 1 GPU): all GPU tests on the new default,
# shuffled timing of the previous build vs SV_SFX_SHADOW=0/1, a short bench
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/pytest_sfx.log; cat gpurun_out/pytest_sfx.log
SV_ROUNDS=15 timeout 600 python scripts/time_variants.py variants/lib_old.so variants/lib_sf0.so variants/lib_sf1.so > gpurun_out/sfx_variants.log 2>&1; tail -5 gpurun_out/sfx_variants.log
SV_BH=16 SV_ROUNDS=15 timeout 600 python scripts/time_variants.py variants/lib_sf0.so variants/lib_sf1.so > gpurun_out/sfx_variants16.log 2>&1; tail -4 gpurun_out/sfx_variants16.log
timeout 600 python bench.py > gpurun_out/bench_sfx.log 2>&1; tail -1 gpurun_out/bench_sfx.log
