# round-end measurement set: full GPU suite, bench lines C1-C5 + reference arm, C3 ncu launch list
mkdir -p gpurun_out/r2f
PYTHONUNBUFFERED=1 timeout -s KILL 1500 python -m pytest tests -v -m gpu -p no:cacheprovider --timeout=600 > gpurun_out/r2f/gputest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/r2f/gputest.log
timeout 900 python bench.py > gpurun_out/r2f/bench_c3.log 2>&1; echo c3=$?
timeout 600 python bench.py --impl reference > gpurun_out/r2f/bench_ref.log 2>&1; echo ref=$?
timeout 300 python bench.py --config c1 --no-cpu > gpurun_out/r2f/bench_c1.log 2>&1
timeout 300 python bench.py --config c2 --no-cpu > gpurun_out/r2f/bench_c2.log 2>&1
timeout 600 python bench.py --config c4 > gpurun_out/r2f/bench_c4.log 2>&1
timeout 600 python bench.py --config c5 > gpurun_out/r2f/bench_c5.log 2>&1
python tools/ncu_target.py c3 > gpurun_out/r2f/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2f/launches_c3.csv python tools/ncu_target.py c3 > gpurun_out/r2f/ncu.log 2>&1; echo ncu=$?; gzip -f gpurun_out/r2f/launches_c3.csv
