for v in 0 1 2 3; do
  echo "== variant $v"; LFGPU_ATTN_VARIANT=$v python -m pytest tests/test_gpu_encoder.py -x -q -k attention 2>&1 | tail -1
  LFGPU_ATTN_VARIANT=$v python tools/encoder_latency.py 2>&1 | grep "packed 64"
done
