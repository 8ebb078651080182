python -c "import __graft_entry__ as g; g.build()"
timeout 120 python scripts/prof_attn.py csla 2 > gpurun_out/dbg1.log 2>&1
timeout 120 compute-sanitizer --tool memcheck python scripts/prof_attn.py csla 1 > gpurun_out/dbg2.log 2>&1
head -50 gpurun_out/dbg1.log; head -60 gpurun_out/dbg2.log
