#!/bin/bash
# Quick C5 headline check (no e2e, no CPU baseline, no C4): value, update/partition ms
python bench.py --no-e2e --no-cpu-baseline --c4-tiles 0 2>/dev/null | python -c "
import json, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
r = d['roofline']
print('C5 value', round(d['value'], 1), 'update_ms', round(r['update_ms'], 4), 'partition_ms', round(r['partition_ms'], 4),
      'other', {k: round(v['value'], 2) for k, v in (d.get('other_configs') or {}).items()})"
