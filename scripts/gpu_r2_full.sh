# Round-2: tests, bench line, C5 workload, sanitizer pass
mkdir -p gpurun_out
timeout 300 python scripts/sanitize_suite.py > gpurun_out/san_plain.log 2>&1; echo RC=$? >> gpurun_out/san_plain.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --target-processes all --print-limit 50 python scripts/sanitize_suite.py > gpurun_out/san_$tool.log 2>&1; echo RC=$? >> gpurun_out/san_$tool.log
done
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest.log 2>&1; echo PYTEST=$? >> gpurun_out/pytest.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo BENCH=$? >> gpurun_out/bench.err
timeout 600 python bench.py --workload c5 --steps 20 --warmup 5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo BENCH=$? >> gpurun_out/bench_c5.err
echo DONE
