set -u
timeout 600 python bench.py --no-cpu-baseline --no-e2e > /tmp/b.json 2>/dev/null; python -c "
import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('value', d['value'], 'e_total', repr(d['e_total']), {k:round(v,4) for k,v in d['phases_ms'].items()})"
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_forces.py -q -m gpu -k "golden or headline or config or random or forces_match or moment" 2>&1 | tail -2
