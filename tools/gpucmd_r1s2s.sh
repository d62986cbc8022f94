timeout 300 python tools/prof_mlmv.py
timeout 300 python tools/prof_gram.py
