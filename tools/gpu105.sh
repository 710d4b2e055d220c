timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2v105.log 2>&1; echo rc=$? >> gpurun_out/smoke_r2v105.log
timeout 1500 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider > gpurun_out/pytest_r2v105.log 2>&1; echo rc=$? >> gpurun_out/pytest_r2v105.log
timeout 1500 python bench.py > gpurun_out/bench_r2v105.log 2>&1; echo rc=$? >> gpurun_out/bench_r2v105.log
