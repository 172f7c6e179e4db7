# ncu launch list of a few device iterations of a config ($1), after the plain run exits 0
python profiles/solve_iters.py $1 3 > gpurun_out/plain_$1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_$1.csv \
    python profiles/solve_iters.py $1 3 > gpurun_out/ncu_launch_$1.log 2>&1
