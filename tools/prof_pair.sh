timeout 300 python -m pytest tests/test_gpu_pair.py -q 2>&1 | tail -2
for c in "128 1" "128 2"; do set -- $c
LFGPU_PAIR_BN=$1 LFGPU_PAIR_S=$2 TRACE_COLD=1 timeout 120 python tools/pair_trace.py 1024 2>&1 | head -9
done
timeout 100 python tools/gemm_ceiling.py 4096 8192 | cut -c1-250
for cfg in "256 1" "256 2" "128 1" "128 2" "128 4" "64 2"; do set -- $cfg;
  LFGPU_PAIR_BN=$1 LFGPU_PAIR_S=$2 timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pair_kernel|umma_kernel" -c 8 --csv python tools/gemm_ceiling.py 1024 --bk --reps 4 2>/dev/null | grep gpu__time | awk -F, -v c="$1/$2" '{print c, $NF}' | tail -1
done
