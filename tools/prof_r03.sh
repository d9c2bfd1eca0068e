# final-round ncu evidence for the cfg2 GEMM (one GPU): launch list with DRAM
# bytes, then one --set full capture. Outputs under gpurun_out/.
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/r03_launches.csv python tools/profile_kernels.py gemm_bench_r03 conv_b1r02 conv_b16r02 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:umma_kernel -s 2 -c 1 \
    -o gpurun_out/r03_gemm_bench python tools/profile_kernels.py gemm_bench_r03 > /dev/null 2>&1
ls -la gpurun_out/r03*
