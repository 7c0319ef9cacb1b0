set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import paper_2403_06218_b200 as T; T.lib(); print('lib ok')"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -20
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -40
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -5
