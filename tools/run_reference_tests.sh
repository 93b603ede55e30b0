#!/usr/bin/env bash
# Runs the reference's own hot-path test files, UNCHANGED, against the B200
# package on a GPU box (VERDICT r1 missing #4).  Run it HERE (it reads
# /root/reference, which the GPU box does not have): the test files travel
# inside the gpurun command as an xz tarball, are unpacked under /tmp on the
# box, and import the package through tools/refshim/lidarseg (the reference's
# package name).  Nothing is copied into the repo; the log lands in
# gpurun_out/reftests.log (profiles/r02/reference_tests.log is a copy).
#
#   bash tools/run_reference_tests.sh
set -euo pipefail
files="conftest.py test_scan.py test_mesh.py test_normals.py test_segment.py test_simulate.py test_evaluate.py"
blob=$(tar -C /root/reference/pkg/tests -cJf - $files | base64 -w0)
exec /usr/local/graft/bin/gpurun --timeout 1200 -- "mkdir -p gpurun_out /tmp/lidarseg_reftests && \
echo $blob | base64 -d | tar -C /tmp/lidarseg_reftests -xJf - && \
PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=\$GRAFT_REPO_ROOT/tools/refshim:\$GRAFT_REPO_ROOT \
timeout 1000 python -m pytest -p no:cacheprovider -v -rA /tmp/lidarseg_reftests > gpurun_out/reftests.log 2>&1; \
rc=\$?; tail -3 gpurun_out/reftests.log; exit \$rc"
