#!/bin/bash
# One parametrised runner for the GPU box (run under gpurun, 1 GPU):
#   gpurun --timeout 1800 -- 'bash scripts/gpu.sh test smoke bench launches'
# Tasks (run in the order given; each writes gpurun_out/<task>.log):
#   test       pytest -m gpu
#   smoke      __graft_entry__.smoke()
#   bench      python bench.py (driver defaults)                    -> gpurun_out/bench.log
#   bench2b    python bench.py --config 2b
#   launches   ncu launch list of the bench command (gpu__time_duration, clocks unlocked)
#   ncu:<regex>[:<bench args>]  one `ncu --set full` capture of the first launch matching <regex>
#   sanitize   compute-sanitizer memcheck / racecheck / synccheck / initcheck on tiny and 256eq
#   sweep      scripts/sweep.py                                     -> gpurun_out/sweep.jsonl
#   py:<script> [args...] via SVARGS env    python scripts/<script>
set -x
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
for t in "$@"; do
  case "$t" in
    test)
      timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/test.log
      cat gpurun_out/test.log ;;
    smoke)
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
      tail -3 gpurun_out/smoke.log ;;
    bench)
      timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -2 gpurun_out/bench.log ;;
    bench2b)
      timeout 900 python bench.py --config 2b > gpurun_out/bench2b.log 2>&1
      tail -2 gpurun_out/bench2b.log ;;
    launches)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 \
        --no-cpu-baseline > gpurun_out/launches.log 2>&1
      tail -1 gpurun_out/launches.log ;;
    ncu:*)
      IFS=: read -r _ rx bargs <<< "$t"
      tag=$(echo "$rx" | tr -c 'a-zA-Z0-9_' '_')
      timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$rx" -s 2 -c 1 \
        --metrics sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active \
        -f -o gpurun_out/ncu_$tag python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
        $bargs > gpurun_out/ncu_$tag.log 2>&1
      tail -3 gpurun_out/ncu_$tag.log ;;
    sanitize)
      for cfg in tiny 256eq; do
        for tool in memcheck racecheck synccheck initcheck; do
          timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py $cfg \
            > gpurun_out/sanitize_${tool}_${cfg}.log 2>&1
          echo "$tool $cfg: exit $? $(tail -1 gpurun_out/sanitize_${tool}_${cfg}.log)"
        done
      done ;;
    sweep)
      timeout 1200 python scripts/sweep.py > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
      tail -3 gpurun_out/sweep.jsonl ;;
    py:*)
      s=${t#py:}
      timeout 1200 python scripts/$s $SVARGS > gpurun_out/${s%.py}.log 2>&1
      tail -5 gpurun_out/${s%.py}.log ;;
  esac
done
