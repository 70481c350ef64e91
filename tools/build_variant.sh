# build a tuning variant of the library: tools/build_variant.sh NAME "-DSLM_STAGE=25760 -DSLM_NS=3"
set -e
D=paper_2409_12892_b200
mkdir -p $D/_variants/$1
for f in raster residuals cache jtj stream pcg; do
  nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -I include --expt-relaxed-constexpr $2 -c $D/csrc/$f.cu -o $D/_variants/$1/$f.o
done
nvcc -shared -gencode arch=compute_100a,code=sm_100a $D/_variants/$1/*.o -o $D/_variants/$1/libsplatlm_b200.so
