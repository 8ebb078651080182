for lib in prev emu0; do
SPARVAR_LIB=variants/lib_$lib.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 -o gpurun_out/ncu_$lib -f python scripts/prof_attn.py csla 3 > gpurun_out/ncu_$lib.log 2>&1
done
