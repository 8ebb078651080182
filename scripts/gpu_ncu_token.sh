# ncu evidence for the NEXT(2) token kernels and the NEXT(3) fused pass (run under gpurun; 1 GPU)
python -c "import __graft_entry__ as g; g.build()"
ncu --set full --import-source on --clock-control none -k regex:"colsum_kernel|token_attn_kernel|topk_tokens|map_tokens" -c 4 \
    -o gpurun_out/token_full -f python scripts/token_bench.py --reps 1 > gpurun_out/ncu_token.log 2>&1
tail -2 gpurun_out/ncu_token.log
