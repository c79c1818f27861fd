set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
timeout 900 python -m pytest tests/test_gpu_evict.py -x -q ${EVICT_K:+-k "$EVICT_K"} 2>&1 | tail -40
