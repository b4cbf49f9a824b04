for l in 5 2 1 0; do echo "LTPO=$l"; QF_GATHER_LTPO=$l QF_ENGINE=resident python tools/profile_case.py C4 3 2 2>&1 | tail -1 | grep -o "'resident_ms': [0-9.]*"; done
