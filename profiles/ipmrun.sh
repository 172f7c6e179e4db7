# IPM A/B: tests on the default library, phase profile of each library given
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/clk.txt
python -m pytest tests/test_gpu_solver.py tests/test_gpu_properties.py tests/test_gpu_integration.py -x -q -k "ipm" -p no:cacheprovider > gpurun_out/t_ipm.log 2>&1
for lib in "$@"; do
  echo "== $lib" >> gpurun_out/ipmprof.log
  USBS_LIB=$lib USBS_IPM_PROF=1 python profiles/prof_kernels.py ipm >> gpurun_out/ipmprof.log 2>&1
done
