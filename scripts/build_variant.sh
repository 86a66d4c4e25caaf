# usage: scripts/build_variant.sh NAME "-DFLAGS ..."  -> build/var/libcc_NAME.so
n=$1; f=$2; mkdir -p build/var/$n
for src in paper_2008_03909_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $f -c $src -o build/var/$n/$(basename $src .cu).o &
done; wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared build/var/$n/*.o -o build/var/libcc_$n.so -lcudart
