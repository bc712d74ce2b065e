mkdir -p gpurun_out/r02
python -m pytest tests/test_gpu_frame.py -q -x -k "kfr" > gpurun_out/r02/t14.log 2>&1
for cfg in "4 2 3 256" "4 3 3 256" "4 2 3 384"; do set -- $cfg; SSS_KFR_STEPS=$1 SSS_KFR_SLOTS=$2 SSS_KFR_MINB=$3 SSS_KFR_CHUNK=$4 python tools/transfer_ab.py kfr | sed "s/^/$1-$2-$3-$4 /" >> gpurun_out/r02/ab14.json 2>> gpurun_out/r02/ab14.err; done
