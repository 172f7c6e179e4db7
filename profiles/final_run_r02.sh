set -x
(time python -m pytest tests -m gpu -x -q) > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
python profiles/configs.py C1 C2 C5 C4 --iters 100000 --budget 200 > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
bash profiles/launches_r02.sh
python profiles/configs.py C3 --iters 100000 --budget 900 >> gpurun_out/configs.jsonl 2>> gpurun_out/configs.err
