# ncu --set full captures of the kernels changed in round 2 (second half)
ncu --set full --import-source on --clock-control none -k regex:k_spmm_g --launch-count 1 -o gpurun_out/spmm_g_c4 python profiles/spmm_one.py 11 C4 > gpurun_out/ncu_spmm.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_compressed_mma_pipe --launch-count 1 -o gpurun_out/k4_c4 python profiles/k4_one.py C4 > gpurun_out/ncu_k4c4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_compressed_mma_pipe --launch-count 1 -o gpurun_out/k4_c5 python profiles/k4_one.py C5 > gpurun_out/ncu_k4c5.log 2>&1
