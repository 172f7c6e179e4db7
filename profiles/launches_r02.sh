# ncu launch list of the bench command (C4), after the same command exits 0 without ncu
python bench.py --steps 2 --warmup 3 --no-cpu --context 0 --ttg-budget 0 --opapply 0 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --context 0 --ttg-budget 0 --opapply 0 > gpurun_out/ncu_launch.log 2>&1
