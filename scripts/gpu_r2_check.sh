# Round-2 iteration: GPU tests (new parity file first), bench line.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity_bench.py -q -x > gpurun_out/pytest_new.log 2>&1; echo PYTEST_NEW=$? >> gpurun_out/pytest_new.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest.log 2>&1; echo PYTEST=$? >> gpurun_out/pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo BENCH=$? >> gpurun_out/bench.err
echo DONE
