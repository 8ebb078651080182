# full-set ncu capture of the bench's CSLA attention launch and predictor (run under gpurun; 1 GPU)
python -c "import __graft_entry__ as g; g.build()"
ncu --set full --import-source on --clock-control none -k regex:"attn_fwd_kernel" -s 2 -c 1 \
    -o gpurun_out/final_attn -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_final_attn.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"predict_kernel" -s 2 -c 1 \
    -o gpurun_out/final_pred -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_final_pred.log 2>&1
tail -n 1 gpurun_out/ncu_final_attn.log; tail -n 1 gpurun_out/ncu_final_pred.log
