timeout 900 python -m pytest tests/test_bands.py -q -x -p no:cacheprovider > gpurun_out/r2l_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2l_pytest.log
python scripts/band_mp1.py c2 > gpurun_out/r2l_band.txt 2>&1
python scripts/band_mp1.py c5 >> gpurun_out/r2l_band.txt 2>&1
