python -c "import __graft_entry__ as g; g.build()"
ncu --set full --import-source on --clock-control none -k regex:"predict" -c 1 -o gpurun_out/pred_full -f python scripts/prof_attn.py pred 1 > gpurun_out/ncu_pred.log 2>&1
tail -3 gpurun_out/ncu_pred.log
