for z in 4 8 16; do
echo "ZDBG=$z" >> gpurun_out/zdbg_r2v76.log
KFBI_ZDBG=$z timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --tb=line -p no:cacheprovider -k "runs_1024_vs_oracle_window and heat" >> gpurun_out/zdbg_r2v76.log 2>&1
done
