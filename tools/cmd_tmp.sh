python tools/polar_stats.py C4 3 resident
QF_ENGINE=resident python tools/profile_case.py C4 3 2 2>&1 | tail -1 | grep -o "'resident_ms': [0-9.]*"
python -m pytest tests -m gpu -x -q -k "resident or RESIDENT or random or C4" 2>&1 | tail -2
