python -m pytest tests/test_gpu_k1_lanczos.py tests/test_gpu_fullscale.py -x -q -p no:cacheprovider > gpurun_out/t_spmm.log 2>&1
python profiles/spmm_ab.py C4 > gpurun_out/spmm_ab.log 2>&1
python bench.py --steps 10 --warmup 3 --context 0 --ttg-budget 0 --no-cpu > gpurun_out/bench_short.log 2>&1
