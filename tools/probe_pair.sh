for cfg in "256 1" "256 2" "256 4" "128 2"; do
  set -- $cfg
  echo "BN=$1 S=$2 bk: $(LFGPU_PAIR_BN=$1 LFGPU_PAIR_S=$2 python tools/gemm_ceiling.py 1024 --factors 256 64 256 --tile $1 --bk --reps 50 2>&1 | tail -1 | cut -c60-230)"
done
LFGPU_PAIR_BN=256 LFGPU_PAIR_S=2 timeout 120 python -m pytest tests/test_gpu_pair.py -q -x 2>&1 | tail -2
