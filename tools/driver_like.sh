#!/bin/bash
# What the round-end driver runs, on a 2-GPU box: tests, smoke, bench N=1, torchrun N=2, reference arm N=1/N=2.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo build=$?
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > /tmp/b1.json 2>/dev/null; echo bench1=$?; wc -l < /tmp/b1.json
timeout 900 python bench.py --impl reference > /tmp/r1.json 2>/dev/null; echo ref1=$?; wc -l < /tmp/r1.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 > /tmp/b2.json 2>/dev/null; echo bench2=$?; wc -l < /tmp/b2.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --impl reference --gpus 2 > /tmp/r2.json 2>/dev/null; echo ref2=$?; wc -l < /tmp/r2.json
python - <<'P'
import json
for f in ['/tmp/b1.json', '/tmp/r1.json', '/tmp/b2.json', '/tmp/r2.json']:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d.get('impl', 'ours'), d['n_gpus'], round(d['ms_per_step'], 3), '%.3e' % d['value'], d.get('e2e', {}).get('value'), d.get('gpu_launches'))
P
