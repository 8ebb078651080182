python -c "import __graft_entry__ as g; g.build()"
for lib in nosmload nsnl_sl100 sl20 sl100; do SPARVAR_LIB=variants/lib_$lib.so timeout 120 python scripts/prof_attn.py pred 20 | sed "s/^/$lib /"; done
timeout 120 python scripts/prof_attn.py pred 20 | sed "s/^/split /"
