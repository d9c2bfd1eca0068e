timeout 300 ncu --set full --clock-control none --import-source on -k regex:umma_kernel -s 2 -c 1 -o gpurun_out/prof_conv_trans python tools/profile_kernels.py conv_trans > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:umma_kernel -s 4 -c 1 -o gpurun_out/prof_bert_gemm python tools/plan_once.py bert 1 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
