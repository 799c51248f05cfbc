# Build libmcg from a commit's sources into _lib/exp_NAME (same-call A/B of
# two versions). Usage: bash profiles/scripts/build_commit.sh NAME COMMIT
set -e
cd "$(dirname "$0")/../.."
T=$(mktemp -d)
mkdir -p $T/a/b/csrc $T/a/include
for f in $(git ls-tree --name-only $2 paper_2305_07238_b200/csrc/); do git show $2:$f > $T/a/b/csrc/$(basename $f); done
git show $2:include/mcg.h > $T/a/include/mcg.h
L=paper_2305_07238_b200/_lib/exp_$1
mkdir -p $L
JI=$(python -c "import sys; sys.path.insert(0,'paper_2305_07238_b200'); import build; print(build.json_include())")
for cu in $T/a/b/csrc/*.cu; do
  nvcc -ccbin /usr/bin/g++ -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo --fmad=false \
    -Xcompiler -fPIC,-ffp-contract=off -I$T/a/include -c $cu -o $L/$(basename $cu).o > /dev/null 2>&1 &
done
for cpp in $T/a/b/csrc/*.cpp; do
  /usr/bin/g++ -std=c++20 -O2 -ffp-contract=off -fPIC -g0 -I$JI -I$T/a/include -c $cpp -o $L/$(basename $cpp).o &
done
wait
nvcc -ccbin /usr/bin/g++ -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $L/libmcg.so $L/*.o \
  -Xcompiler -fPIC -lpthread
echo built $L/libmcg.so
