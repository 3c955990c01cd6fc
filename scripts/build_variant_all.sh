# Build libss_b200_NAME.so with extra -D flags on EVERY source (knobs in problem.h such as SSB_KDENSE
# change the setup's layout as well as the kernel).  usage: bash scripts/build_variant_all.sh NAME "-DSSB_X=1 ..."
set -e
cd "$(dirname "$0")/../paper_1411_4356_b200/csrc"
NAME=$1; FLAGS=$2
mkdir -p obj_$NAME
for f in build spmv trsv krylov solution; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -Xcompiler -ffp-contract=off --expt-relaxed-constexpr $FLAGS -c $f.cu -o obj_$NAME/$f.o &
done
for f in capi setup rcm ilut; do
  g++ -O2 -std=c++17 -fPIC -ffp-contract=off -pthread -I/usr/local/cuda/include $FLAGS -c $f.cpp -o obj_$NAME/$f.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libss_b200_$NAME.so obj_$NAME/*.o \
  -Xcompiler -pthread -lcudart_static -lrt -ldl
echo built ../libss_b200_$NAME.so
