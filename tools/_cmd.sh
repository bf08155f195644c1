timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_full.log 2>&1; echo pytest=$? >> gpurun_out/pytest_full.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench=$? >> gpurun_out/smoke.log
