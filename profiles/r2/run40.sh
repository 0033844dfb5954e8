python profiles/e2e_only.py 3 2>&1 | tail -3
