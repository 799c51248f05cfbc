# Build an experimental libmcg variant: every .cu recompiled with extra nvcc
# flags, linked with the normal build's host objects.
# Usage: bash profiles/scripts/build_variant.sh NAME "-DFOO=1 ..."
# Load it with MCG_LIB_PATH=paper_2305_07238_b200/_lib/exp_NAME/libmcg.so
set -e
cd "$(dirname "$0")/../.."
python paper_2305_07238_b200/build.py > /dev/null
L=paper_2305_07238_b200/_lib
mkdir -p $L/exp_$1
: > $L/exp_$1/ptxas.log
for cu in paper_2305_07238_b200/csrc/*.cu; do
  b=$(basename $cu)
  nvcc -ccbin /usr/bin/g++ -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo --fmad=false \
    -Xptxas -v -Xcompiler -fPIC,-ffp-contract=off -Iinclude $2 \
    -c $cu -o $L/exp_$1/$b.o >> $L/exp_$1/ptxas.log 2>&1 &
done
wait
objs=$(ls $L/obj/*.o | grep -v "\.cu\.o")
nvcc -ccbin /usr/bin/g++ -gencode arch=compute_100a,code=sm_100a -shared -cudart static \
  -o $L/exp_$1/libmcg.so $objs $L/exp_$1/*.cu.o -Xcompiler -fPIC -lpthread
echo built $L/exp_$1/libmcg.so
