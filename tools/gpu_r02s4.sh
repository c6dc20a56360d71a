timeout 900 python -m pytest tests/test_bf16_gpu.py -x -q -k "fused_sgd" 2>&1 | tail -n 3
