for p in od qd; do timeout 300 python tools/time_variants.py $p 1024 128 2>&1 | head -2; done
timeout 1200 python -m pytest tests -m gpu -q -x -k "qr or invariants or determinism or sharded or complex" 2>&1 | tail -2
