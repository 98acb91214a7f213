# Quick GPU pass: gpu tests + the default bench line (no profilers).
# Usage (repo root, under gpurun): bash scripts/gpu_quick.sh TAG [pytest-args]
TAG=${1:-q}
shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q "$@" > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-wcrt --no-sim > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json,sys,glob,os
tag=os.environ.get("TAG_Q")
PY
python -c "
import json,sys
l=open('gpurun_out/bench_$TAG.log').read().strip().splitlines()[-1]
d=json.loads(l)
print('main', d['value'], 'e2e', d['e2e']['value'], 'stage_ms', d['roofline']['stage_ms'])
for k,v in d.get('workloads',{}).items():
    print(k, v.get('value'), v.get('stage_ms'), v.get('stage_sets'), v.get('parity'), v.get('error'))
"
