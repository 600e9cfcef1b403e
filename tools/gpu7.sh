for n in 53 128 256; do timeout 300 python tools/cg_micro.py $n 1000; done 2>&1 | grep -v Warn
timeout 900 python -m pytest tests -q -m gpu -x --durations=3 2>&1 | tail -6
