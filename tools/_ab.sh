python tools/ab_knobs.py elem_path 0,0 5,3,4 2>&1 | tail -6
