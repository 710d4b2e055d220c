for y in 0 2 3 4 8 12; do
KFBI_SPEC_Y=$y timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"spec_block" -c 6 --csv --log-file gpurun_out/specy${y}_r2v88.csv python bench.py --no-configs --no-slab --no-pipeline-pass --steps 1 --warmup 3 --sequential > /dev/null 2>&1
done
