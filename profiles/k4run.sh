python -m pytest tests/test_gpu_constraints.py tests/test_gpu_solver.py -x -q -k "compressed or constraint" -p no:cacheprovider > gpurun_out/t_k4.log 2>&1
python profiles/k4_time.py C4 C5 C3 > gpurun_out/k4.log 2>&1
