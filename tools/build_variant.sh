# build paper_1104_3349_b200/libmscg_<name>.so with extra nvcc flags for trisolve.cu
# usage: bash tools/build_variant.sh <name> [flags...]
set -e
name=$1; shift
cd "$(dirname "$0")/.."
python -m paper_1104_3349_b200.build > /dev/null
nvcc "$@" -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -Xcompiler -ffp-contract=off --expt-relaxed-constexpr -I include -I paper_1104_3349_b200/csrc -c paper_1104_3349_b200/csrc/device/trisolve.cu -o /tmp/tri_$name.o
objs=$(ls paper_1104_3349_b200/_build/*.o | grep -v device_trisolve)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_1104_3349_b200/libmscg_$name.so $objs /tmp/tri_$name.o -lpthread
echo built libmscg_$name.so
