timeout 1200 compute-sanitizer --tool initcheck --print-limit 50 python tools/sanitize_driver.py > gpurun_out/sanitizer_initcheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitizer_initcheck.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_headline.py -m gpu -q --tb=short -p no:cacheprovider > gpurun_out/pytest_r2v85.log 2>&1; echo rc=$? >> gpurun_out/pytest_r2v85.log
bash tools/gpu84.sh
