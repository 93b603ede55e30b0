# parity tests on the default library, then A/B timing of variants
timeout 900 python -m pytest tests -m gpu -x -q ${TESTS:-} > gpurun_out/gputest.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/gputest.log
bash tools/variants2.sh ${VARIANTS:-base}
