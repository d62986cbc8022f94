timeout 300 python tools/prof_mlmv.py
timeout 300 python tools/prof_gram.py
timeout 300 python tools/trace_tucker.py c3 2>&1 | grep "=="
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
