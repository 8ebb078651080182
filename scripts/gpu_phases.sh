SPARVAR_LIB=variants/lib_prof.so timeout 120 python scripts/prof_phases.py csla
SPARVAR_LIB=variants/lib_prof0.so timeout 120 python scripts/prof_phases.py csla
