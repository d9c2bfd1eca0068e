timeout 600 python -m pytest tests/test_gpu_pair.py -x -q 2>&1 | grep -E "Error|error|assert|FAILED|def test|Mismatch|mismatch" | head -30
LFGPU_PAIR_DIAG=1 LFGPU_PAIR_BN=128 LFGPU_PAIR_S=2 python tools/pair_trace.py 1024 256 64 256 2>&1 | grep -A1 "tile0 chunks" | head -4
