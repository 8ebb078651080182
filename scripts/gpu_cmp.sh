timeout 300 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -2
python scripts/time_variants.py "$@"
