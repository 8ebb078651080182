set -x
python -c "import __graft_entry__ as g; g.build()"
for w in csla cs4a dense; do timeout 120 python scripts/prof_attn.py $w 20; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 -o gpurun_out/prof_v1 -f python scripts/prof_attn.py csla 3 > gpurun_out/ncu_v1.log 2>&1
tail -3 gpurun_out/ncu_v1.log
