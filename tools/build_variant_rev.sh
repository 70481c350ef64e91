# build the library of a git revision as a tuning variant: tools/build_variant_rev.sh NAME REV
set -e
D=paper_2409_12892_b200
T=$(mktemp -d)
git archive $2 $D/csrc include | tar -x -C $T
mkdir -p $D/_variants/$1
for f in raster residuals cache jtj stream pcg; do
  nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -I $T/include --expt-relaxed-constexpr -c $T/$D/csrc/$f.cu -o $D/_variants/$1/$f.o
done
nvcc -shared -gencode arch=compute_100a,code=sm_100a $D/_variants/$1/*.o -o $D/_variants/$1/libsplatlm_b200.so
rm -rf $T
