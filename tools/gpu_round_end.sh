nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/gputests.log 2>&1; echo TESTS_EXIT $? >> gpurun_out/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo SMOKE_EXIT $? >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo BENCH_EXIT $? >> gpurun_out/bench.err
python bench.py --config c4 --no-solve --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-other --no-solve > gpurun_out/ncu.log 2>&1
