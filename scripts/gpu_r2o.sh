# the whole GPU suite on the bounds-checked build (a trap fails the test), then on the default build
mkdir -p gpurun_out/checked
SEEDS_LIB=scripts/alt_checked.so timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/checked/pytest_checked.log 2>&1; echo "exit $?" >> gpurun_out/checked/pytest_checked.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/checked/pytest_default.log 2>&1; echo "exit $?" >> gpurun_out/checked/pytest_default.log
