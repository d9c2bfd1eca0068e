mkdir -p gpurun_out
(for ds in 0 1; do LFGPU_PAIR_DBG_SPLIT=$ds LFGPU_PAIR_BN=256 LFGPU_PAIR_S=2 timeout 60 python tools/pair_debug.py 512 1024 512 128 64 256; done
 BK=1 LFGPU_PAIR_BN=256 LFGPU_PAIR_S=2 timeout 60 python tools/pair_debug.py 512 1024 512 128 64 256) > gpurun_out/pair_debug.log 2>&1
cat gpurun_out/pair_debug.log
