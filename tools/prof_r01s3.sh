# round 1 session 3 captures (run under gpurun from the repo root)
set -x
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r01s3_launches.csv python tools/profile_bench.py all > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:umma_kernel -s 2 -c 1 -o gpurun_out/r01s3_gemm python tools/profile_bench.py gemm > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:umma_kernel -s 2 -c 1 -o gpurun_out/r01s3_conv16 python tools/profile_bench.py conv16 > /dev/null 2>&1
ls -la gpurun_out/r01s3_*
