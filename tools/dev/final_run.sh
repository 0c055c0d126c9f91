# development: the round-end sequence on one GPU (tests, both bench arms, launch list of the bench command)
set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/final_pytest.log
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 1 --warmup 3 --skip-configs > gpurun_out/final_ncu.log 2>&1
cat gpurun_out/final_pytest.log; head -c 400 gpurun_out/final_bench.json; echo; head -c 600 gpurun_out/final_bench_ref.json
