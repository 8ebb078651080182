python -c "import __graft_entry__ as g; g.build()"
timeout 300 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -15
python scripts/time_variants.py variants/lib_prev.so variants/lib_v2.so
SPARVAR_LIB=variants/lib_prof2.so timeout 120 python scripts/prof_phases.py csla 2>&1 | grep -v "^\[\|^ \["
