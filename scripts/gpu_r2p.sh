ALTS="scripts/alt_xp_NOFENCE.so scripts/alt_xp_ISSUER.so" CFGS="c2 c3" bash scripts/gpu_ab.sh > gpurun_out/r2p_ab.txt 2>&1
timeout 600 python -m pytest tests/test_bands.py -q -x -p no:cacheprovider > gpurun_out/r2p_bands.log 2>&1; echo "exit $?" >> gpurun_out/r2p_bands.log
python scripts/band_mp1.py c5 > gpurun_out/r2p_band.txt 2>&1
