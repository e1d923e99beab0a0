python tools/e2eprof.py 2>&1 | head -5
python bench.py --no-cpu-baseline --nrhs-big 0 --no-residual 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], 'e2e', d['e2e']['value'])"
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_boundary.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
