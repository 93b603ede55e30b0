# full ncu capture of named kernels + source / details / raw digests: KERNELS="k_tile k_tile_cc" FRAMES=128
KERNELS="${KERNELS:-k_tile}" FRAMES=${FRAMES:-128} bash tools/r2_ncu.sh
for k in ${KERNELS:-k_tile}; do
ncu -i gpurun_out/prof_$k${TAG:-}.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${k}${TAG:-}_src.csv 2>&1
ncu -i gpurun_out/prof_$k${TAG:-}.ncu-rep --page details > gpurun_out/${k}${TAG:-}_details.txt 2>&1
ncu -i gpurun_out/prof_$k${TAG:-}.ncu-rep --page raw --csv > gpurun_out/${k}${TAG:-}_raw.csv 2>&1
done
