# Build libss_b200_NAME.so: trsv.cu compiled with extra -D flags, linked with the default objects.
# usage: bash scripts/build_variant.sh NAME "-DSSB_X=1 ..."   (run `make` first)
set -e
cd "$(dirname "$0")/../paper_1411_4356_b200/csrc"
NAME=$1; FLAGS=$2
mkdir -p obj_$NAME
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -ffp-contract=off --expt-relaxed-constexpr $FLAGS -c trsv.cu -o obj_$NAME/trsv.o
OBJS=$(ls obj/*.o | grep -v trsv.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libss_b200_$NAME.so $OBJS obj_$NAME/trsv.o \
  -Xcompiler -pthread -lcudart_static -lrt -ldl
echo built ../libss_b200_$NAME.so
