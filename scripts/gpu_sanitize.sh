# compute-sanitizer evidence (memcheck / racecheck / synccheck) on small grid-mode runs
mkdir -p gpurun_out/san
CS=/usr/local/cuda/bin/compute-sanitizer
run() { name=$1; shift; timeout ${TMO:-600} $CS "$@" > gpurun_out/san/$name.txt 2>&1; echo "$name exit $?" >> gpurun_out/san/summary.txt; tail -3 gpurun_out/san/$name.txt >> gpurun_out/san/summary.txt; }
run memcheck_c1 --tool memcheck --leak-check full python scripts/san_case.py cold c1 1 grid
run memcheck_badinit --tool memcheck python scripts/san_case.py badinit
run memcheck_badinit_graph --tool memcheck python scripts/san_case.py badinit c1 1 graph
run memcheck_c2 --tool memcheck python scripts/san_case.py cold c2 1 grid
run memcheck_c3x8 --tool memcheck python scripts/san_case.py cold c3 8 grid
run synccheck_c1 --tool synccheck python scripts/san_case.py cold c1 1 grid
run synccheck_c2 --tool synccheck python scripts/san_case.py cold c2 1 grid
run racecheck_c1 --tool racecheck --racecheck-report all python scripts/san_case.py cold c1 1 grid
run racecheck_c3x8 --tool racecheck --racecheck-report all python scripts/san_case.py cold c3 8 grid
run initcheck_c2 --tool initcheck python scripts/san_case.py cold c2 1 grid
