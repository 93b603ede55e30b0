# parity tests with a given library variant (LSEG_LIB_PATH), then A/B timing of variants
LSEG_LIB_PATH=$PWD/paper_2005_02704_b200/liblidarseg_b200_${TESTLIB}.so timeout 900 python -m pytest tests -m gpu -x -q ${TESTS:-} > gpurun_out/gputest.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/gputest.log
bash tools/variants2.sh ${VARIANTS:-base}
