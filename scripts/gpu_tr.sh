timeout 60 python scripts/trace.py ${CFG:-c2} ${MODE:-grid} 2>&1 | tail -7
