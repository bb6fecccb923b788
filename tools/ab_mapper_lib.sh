# A/B of the mapper (mode 3) between the current library and build/ab/libpkv_b200_pre_f8.so on one box
set -e
mkdir -p /tmp/oldroot/paper_2605_16360_b200
cp paper_2605_16360_b200/*.py /tmp/oldroot/paper_2605_16360_b200/
cp build/ab/libpkv_b200_pre_f8.so /tmp/oldroot/paper_2605_16360_b200/libpkv_b200.so
cp bench.py /tmp/oldroot/
# the tool puts its own parent directory first on sys.path: run the copy so the old library is the one loaded
mkdir -p /tmp/oldroot/tools; cp tools/*.py /tmp/oldroot/tools/
for i in 1 2; do
  python tools/time_mapper_modes.py 3 | sed 's/^/HEAD   /'
  (cd /tmp/oldroot && PYTHONPATH=/tmp/oldroot python /tmp/oldroot/tools/time_mapper_modes.py 3 2>&1 | sed 's/^/pre-F8 /') 
done
