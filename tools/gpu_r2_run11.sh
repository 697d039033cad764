mkdir -p gpurun_out
TAG=r11 bash tools/gpu_r2_iter_noparity.sh
