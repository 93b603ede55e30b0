# A/B the working tree against HEAD on one GPU box: builds HEAD's library as
# the `old` variant (git stash), the working tree as `base`, then (GPU side)
# the parity tests and tools/variants2.sh base old.   bash tools/ab_head.sh [TIMEOUT]
set -e
cd "$(dirname "$0")/.."
if git diff --quiet; then echo "no working-tree changes to compare"; exit 1; fi
git stash -q
python -c "from paper_2005_02704_b200 import _build; _build.build(force=True, out='paper_2005_02704_b200/liblidarseg_b200_old.so')"
git stash pop -q
python -c "from paper_2005_02704_b200 import _build; _build.build(force=True)"
/usr/local/graft/bin/gpurun --timeout ${1:-1500} -- 'timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/gputest.log; bash tools/variants2.sh base old'
rm -f paper_2005_02704_b200/liblidarseg_b200_old.so
