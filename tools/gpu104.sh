for c in 1 0 1; do
KFBI_SPEC_CLUSTER=$c timeout 600 python bench.py --no-configs --no-pipeline-pass --steps 5 --warmup 3 > gpurun_out/bench_cl${c}_r2v104.log 2>&1
python - <<PY >> gpurun_out/c5_cluster_r2v104.txt
import json
d=json.loads([x for x in open('gpurun_out/bench_cl${c}_r2v104.log') if x.startswith('{')][-1])
print("cluster=$c", round(d['value'],1), {k:round(v.get('ms_per_solve',0),1) for k,v in d['slab_c5'].items() if isinstance(v,dict)})
PY
done
