# A/B variants of libmsfm_b200.so with extra -D flags for knn.cu:
#   tools/build_knn_variants.sh NAME "-DFLAG=1 ..." [...]  -> paper_1512_06235_b200/variants/libmsfm_NAME.so
set -e
cd "$(dirname "$0")/../paper_1512_06235_b200/csrc"
make -s >/dev/null
mkdir -p ../variants
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
     -Xcompiler -fPIC -I../../include -fmad=false --expt-relaxed-constexpr -Xptxas -v $flags \
     -c knn.cu -o /tmp/knn_$name.o 2> /tmp/knn_$name.log
  grep -A2 "Function properties for.*knn_tc_kernelILi2ELb1" /tmp/knn_$name.log | grep -i "spill\|regis" | tr '\n' ' '; echo " <- $name"
  objs=$(ls *.o | grep -v '^knn.o$')
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../variants/libmsfm_$name.so \
     /tmp/knn_$name.o $objs -lcudart -Xcompiler -pthread
done
