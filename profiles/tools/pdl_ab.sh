#!/bin/bash
# PDL A/B: AGNN-4 / GCN-2 arxiv epoch (bench.py value) with and without programmatic dependent launch
for pdl in 0 1 0 1; do
  echo -n "TCG_PDL=$pdl: "
  TCG_PDL=$pdl timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('agnn', d['value'], 'e2e', d['e2e']['value'], 'gcn2', d['extras'].get('gcn2_h16_epoch_ms'), 'spmm cold', d['roofline']['launch_us'])"
done
