# Build libcsvgpu.so with extra nvcc flags into variants/NAME.so (A/B timing via CSVGPU_LIB).
# usage: bash tools/build_variant.sh NAME "-DFOO=1 ..."
set -e
mkdir -p variants
cd paper_2308_16619_b200/csrc
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
  -ccbin /usr/bin/g++ --expt-relaxed-constexpr $2 -shared -o ../../variants/$1.so \
  csv_decode.cu csv_encode.cu csv_api.cu csv_cache.cu csv_rans.cu csv_peer.cu -lcudart
