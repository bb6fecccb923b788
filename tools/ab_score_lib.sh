# A/B of scoring pass 1 between the current library and build/ab/libpkv_b200_head.so
# (same box, alternating): tools/time_score.py at the given poly-pair counts.
set -e
mkdir -p /tmp/oldroot/paper_2605_16360_b200
cp paper_2605_16360_b200/*.py /tmp/oldroot/paper_2605_16360_b200/
cp build/ab/libpkv_b200_head.so /tmp/oldroot/paper_2605_16360_b200/libpkv_b200.so
cp bench.py /tmp/oldroot/
# the tool puts its own parent directory first on sys.path: run the copy so the old library is the one loaded
mkdir -p /tmp/oldroot/tools; cp tools/*.py /tmp/oldroot/tools/
for i in 1 2; do
  for p in "$@"; do
    PKV_POLY_PAIRS=$p python tools/time_score.py --iters 3 2>&1 | tail -1 | sed "s/^/new  /"
    (cd /tmp/oldroot && PYTHONPATH=/tmp/oldroot PKV_POLY_PAIRS=$p python /tmp/oldroot/tools/time_score.py --iters 3 2>&1 | tail -1 | sed "s/^/head /")
  done
done
