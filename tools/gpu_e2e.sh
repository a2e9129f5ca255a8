# end-to-end pipeline depth sweep (XLF_E2E_CHUNKS)
for c in 2 3 4; do XLF_E2E_CHUNKS=$c timeout 300 python bench.py --no-cpu --no-blocks > gpurun_out/b.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); print('chunks $c', d['value'], d['e2e'])"; done
