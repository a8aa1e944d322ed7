# Build an experiment variant of libstgmg.so with extra nvcc flags: bash tools/build_variant.sh NAME -DFLAG ...
set -e
name=$1; shift
out=paper_2303_06742_b200/exp/$name; mkdir -p $out
for f in paper_2303_06742_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Iinclude "$@" -c $f -o $out/$(basename $f).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libstgmg.so $out/*.o
echo built $out/libstgmg.so
