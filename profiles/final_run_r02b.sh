# end-of-round evidence: full GPU suite, the default bench line and the reference arm, ncu --set full of the d = 210 IPM
set -x
(time python -m pytest tests -m gpu -x -q) > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
(time python bench.py) > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
(time python bench.py --impl reference) > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
python profiles/ipm_one.py 20 > gpurun_out/ipm_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_ipm --launch-skip 1 --launch-count 1 -o gpurun_out/ipm_d210 python profiles/ipm_one.py 20 > gpurun_out/ncu_ipm.log 2>&1
ls -la gpurun_out/*.ncu-rep
