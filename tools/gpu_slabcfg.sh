timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for c in 0 1; do RHG_SLAB_CFG=$c timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg $c', 'ms',d['ms_per_step'], 'e2e', d['e2e']['value'], 'slab_ms',d['roofline']['kernel_ms'])"; done
