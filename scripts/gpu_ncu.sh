# ncu evidence for the bench command (run under gpurun; 1 GPU).  Writes gpurun_out/.
set -x
python -c "import __graft_entry__ as g; g.build()"
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"attn_fwd|predict" -s 5 -c 3 \
    -o gpurun_out/prof_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
python bench.py --steps 50 --warmup 5 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log
