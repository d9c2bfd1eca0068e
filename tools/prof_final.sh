# round-2 final ncu evidence (one GPU): launch list with DRAM bytes of the
# bench's kernels, then one --set full capture of the cfg2 GEMM. Outputs
# under gpurun_out/.
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/final_launches.csv python tools/profile_kernels.py gemm_bench_final conv_b1r02 conv_b16r02 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:umma_kernel -s 2 -c 1 \
    -o gpurun_out/final_gemm_bench python tools/profile_kernels.py gemm_bench_final > /dev/null 2>&1
ls -la gpurun_out/final*
