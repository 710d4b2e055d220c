set -x
timeout 900 python -m pytest tests/test_gpu_tri.py -m gpu -q --tb=short -p no:cacheprovider -k "facr" > gpurun_out/facr16k_r2v30.log 2>&1; echo rc=$? >> gpurun_out/facr16k_r2v30.log
KFBI_FACR=0 timeout 600 python tools/check_box.py 16384 > gpurun_out/box16k_3p_r2v30.log 2>&1
timeout 600 python tools/check_box.py 16384 8192 4096 > gpurun_out/box16k_facr_r2v30.log 2>&1
