# development check on the GPU box: tests, bench, shard timing (outputs in gpurun_out/$1)
set -u
D=gpurun_out/${1:-check}; mkdir -p $D
timeout 1200 python -m pytest tests -x -q -m gpu > $D/pytest.log 2>&1; tail -3 $D/pytest.log
timeout 600 python bench.py --no-cpu-baseline > $D/bench.json 2> $D/bench.err; python -c "
import json;d=json.load(open('$D/bench.json'));print('value',d['value'],'e2e',d['e2e']['value'],'fixed',d['e2e_fixed_positions']['value'],'phases',{k:round(v,3) for k,v in d['phases_ms'].items()})" || tail -5 $D/bench.err
AB_CONFIG=3 timeout 600 python scripts/shard_timing.py 2>&1 | grep overlap
