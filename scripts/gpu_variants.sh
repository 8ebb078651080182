python -c "import __graft_entry__ as g; g.build()"
timeout 300 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -3
for w in csla cs4a dense; do timeout 120 python scripts/prof_attn.py $w 20; done
for lib in emu0 emu3 emu8; do for w in csla dense; do SPARVAR_LIB=variants/lib_$lib.so timeout 120 python scripts/prof_attn.py $w 20 | sed "s/^/$lib /"; done; done
SPARVAR_LIB=variants/lib_prof0.so timeout 120 python scripts/prof_phases.py csla 2>&1 | head -3
