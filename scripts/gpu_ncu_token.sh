# ncu evidence for the NEXT(2) token kernels (run under gpurun; 1 GPU): one full-set capture each
python -c "import __graft_entry__ as g; g.build()"
for k in colsum_kernel token_attn_kernel topk_tokens_kernel map_tokens_kernel; do
  ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 \
      -o gpurun_out/tok_$k -f python scripts/token_bench.py --reps 1 > gpurun_out/ncu_$k.log 2>&1
  tail -1 gpurun_out/ncu_$k.log
done
