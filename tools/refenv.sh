# Source this to import the read-only reference (vecsym) in THIS container only.
export PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests${PYTHONPATH:+:$PYTHONPATH}
export NUMBA_CACHE_DIR=/tmp/numba_cache
export PYTHONDONTWRITEBYTECODE=1
