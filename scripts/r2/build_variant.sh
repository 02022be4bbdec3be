# A/B build: libvp_<tag>.so with extra nvcc flags (e.g. -DVP_PAIR_WARPS=8); load it with VP_LIB=<path>
# usage: bash scripts/r2/build_variant.sh <tag> <flags...>
set -e
tag=$1; shift
C=paper_2409_11998_b200/csrc
T=$(mktemp -d)
for s in vp_api vp_nufft vp_local vp_levels vp_fft vp_boundary vp_layer vp_bie; do
  nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr "$@" -c $C/$s.cu -o $T/$s.o &
done
wait
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o paper_2409_11998_b200/libvp_$tag.so $T/*.o -lcufft
rm -rf $T
echo paper_2409_11998_b200/libvp_$tag.so
