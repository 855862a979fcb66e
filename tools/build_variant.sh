# Build an A/B variant of libcbspmv.so into ab/<name>/ with extra nvcc flags for kernels.cu
# (optionally from another kernels.cu):  bash tools/build_variant.sh NAME "-DCBSPMV_AGG_BATCH=8" [kernels.cu]
set -e
name=$1; flags=$2; src=${3:-paper_2605_18515_b200/csrc/kernels.cu}
C=paper_2605_18515_b200/csrc
mkdir -p ab/$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v -Iinclude -I$C \
  --expt-relaxed-constexpr $flags -c -o ab/$name/kernels.o $src 2> ab/$name/ptxas.log || (cat ab/$name/ptxas.log; false)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ab/$name/libcbspmv.so $C/builder.o $C/stream.o $C/capi.o $C/mmio.o \
  $C/container.o ab/$name/kernels.o $C/gpu_builder.o $C/exchange.o -lcudart -lpthread
grep -E "Used [0-9]+ registers" ab/$name/ptxas.log | sort | uniq -c | head -3
grep -E "spill" ab/$name/ptxas.log | grep -v " 0 bytes spill stores" | head -3 || true
