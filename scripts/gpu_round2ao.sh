set -u
O=gpurun_out/r02ao; mkdir -p $O
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; python -c "
import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); print('value', d['value'], 'e2e', d['e2e']['value'], 'forces', d['forces_e2e'], d['clocks'])"
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err; python -c "
import json; d=json.loads(open('$O/bench_c4.json').read().strip().splitlines()[-1]); print('value', d['value'], 'e2e', d['e2e']['value'], 'forces', d['forces_e2e'], d['clocks'])"
timeout 900 python -m pytest tests/test_forces.py -q -m gpu -x -k "at_scale or half_shell" 2>&1 | tail -3
