mkdir -p gpurun_out/r02
python -m pytest tests -m gpu -x -q > gpurun_out/r02/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r02/gpu_tests.log
python tools/transfer_ab.py kfr flat16 > gpurun_out/r02/ab.json 2> gpurun_out/r02/ab.err
SSS_KFR_CHUNK=256 python tools/transfer_ab.py kfr > gpurun_out/r02/ab256.json 2>> gpurun_out/r02/ab.err
python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/r02/bench.json 2> gpurun_out/r02/bench.err
