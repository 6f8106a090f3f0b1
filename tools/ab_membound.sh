set -x
python -m pytest tests/test_parity_gpu.py -x -q -k "shapes or outputs_in_bf16 or gqa or bias" 2>&1 | tail -3
for i in 1 2; do
 (cd .ab_old && python bench.py --sweep membound --steps 10 --warmup 3 > ../gpurun_out/mbA$i.jsonl 2>/dev/null)
 python bench.py --sweep membound --steps 10 --warmup 3 > gpurun_out/mbB$i.jsonl 2>/dev/null
done
for f in gpurun_out/mb[AB]?.jsonl; do echo $f; python -c "
import json,sys
for l in open('$f'):
  try: d=json.loads(l)
  except: continue
  print(d.get('config'), d.get('kernels_ms'))
"; done
