# r02 ncu evidence (one GPU): launch list of the benchmarked kernels, then
# one --set full capture of each top kernel. Outputs under gpurun_out/.
set -x
K="gemm_bench gemm_pair conv_b1r02 conv_b16r02 transform"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/r02_launches.csv python tools/profile_kernels.py $K > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:umma_kernel -s 2 -c 1 \
    -o gpurun_out/r02_gemm_bench python tools/profile_kernels.py gemm_bench > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 2 -c 1 \
    -o gpurun_out/r02_gemm_pair python tools/profile_kernels.py gemm_pair > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:umma_kernel -s 2 -c 1 \
    -o gpurun_out/r02_conv_b16 python tools/profile_kernels.py conv_b16r02 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:digit -s 2 -c 1 \
    -o gpurun_out/r02_transform python tools/profile_kernels.py transform > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
