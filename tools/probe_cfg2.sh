set -x
for f in "256 64 256" "256 64 128" "256 64 64" "128 64 128" "256 512 512"; do
  for t in 64 128 256; do
    python tools/gemm_ceiling.py 1024 --factors $f --tile $t --reps 50 2>&1 | tail -1
  done
done
for s in 1 2 4; do LFGPU_PAIR_S=$s python tools/gemm_ceiling.py 1024 --factors 256 64 256 --tile 256 --reps 50 2>&1 | tail -1; done
for s in 1 2 4; do LFGPU_PAIR_S=$s python tools/gemm_ceiling.py 1024 --factors 256 64 128 --tile 128 --reps 50 2>&1 | tail -1; done
LFGPU_NO_PAIR=1 python tools/gemm_ceiling.py 1024 --factors 128 64 128 --tile 128 --reps 50 2>&1 | tail -1
python tools/gemm_ceiling.py 1024 2048 4096 --factors 256 64 256 --tile 256 --reps 50 2>&1 | tail -3
python tools/pair_trace.py 1024 256 64 256 2>&1 | tail -30
LFGPU_PAIR_S=4 python tools/pair_trace.py 1024 256 64 256 2>&1 | tail -30
python tools/pair_trace.py 1024 256 512 512 2>&1 | tail -30
