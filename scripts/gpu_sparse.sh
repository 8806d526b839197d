set -x
export FETI_DEBUG_SYNC=${FETI_DEBUG_SYNC:-1}
timeout 900 python -m pytest tests/test_gpu_sparse.py -x -q -k "not config5" 2>&1 | tail -30
timeout 600 python -m pytest tests/test_gpu_sparse.py -x -q -k "config5" 2>&1 | tail -15
