# 1-CTA kernel: TMA producer warp count vs per-launch time (diagnostics)
for np in 3 5; do
  echo "NP=$np"
  LFGPU_UMMA_NP=$np LFGPU_NO_PAIR=1 python tools/gemm_ceiling.py 1024 --factors 128 64 64 --tile 64 --reps 50 2>&1 | tail -1 | cut -c1-200
  LFGPU_UMMA_NP=$np python tools/chain_probe.py 2>&1 | tail -2
done
