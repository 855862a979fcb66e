# Build every native artefact in-tree (the .so files travel to the GPU box with
# the gpurun snapshot; they are git-ignored).
#   synth/libsynth.so                  seeded input generators (shared by tests + bench)
#   oracle/liboracle.so                plain C oracle (test infrastructure only)
#   paper_2605_18515_b200/libcbspmv.so the C-ABI library: host builder + sm_100a kernels

NVCC      ?= nvcc
CC        ?= gcc
CXX       ?= g++
ARCH      := -gencode arch=compute_100a,code=sm_100a
CUDA_HOME ?= /usr/local/cuda

PKG       := paper_2605_18515_b200
CSRC      := $(PKG)/csrc
LIB       := $(PKG)/libcbspmv.so

ABLATION  ?= 0   # 1: profiling build honouring CBSPMV_DEBUG_SKIP
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall \
             -Xptxas -v -Iinclude -I$(CSRC) --expt-relaxed-constexpr -DCBSPMV_ABLATION=$(ABLATION)
CXXFLAGS  := -O3 -std=c++17 -fPIC -Wall -Wextra -Iinclude -I$(CSRC) -I$(CUDA_HOME)/include -pthread

all: synth oracle lib

synth: synth/libsynth.so
oracle: oracle/liboracle.so
lib: $(LIB)

synth/libsynth.so: synth/synth.c
	$(CC) -O3 -fPIC -shared -Wall -pthread -o $@ $<

oracle/liboracle.so: oracle/oracle.c
	$(CC) -O2 -fPIC -shared -Wall -Wextra -std=c11 -o $@ $<

HOST_OBJS := $(CSRC)/builder.o $(CSRC)/stream.o $(CSRC)/capi.o $(CSRC)/mmio.o $(CSRC)/container.o

$(CSRC)/%.o: $(CSRC)/%.cpp $(CSRC)/cb_internal.h include/cbspmv.h
	$(CXX) $(CXXFLAGS) -c -o $@ $<

$(CSRC)/kernels.o: $(CSRC)/kernels.cu $(CSRC)/cb_internal.h include/cbspmv.h
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $(CSRC)/ptxas.log || (cat $(CSRC)/ptxas.log; false)

$(CSRC)/gpu_builder.o: $(CSRC)/gpu_builder.cu $(CSRC)/cb_internal.h include/cbspmv.h
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $(CSRC)/ptxas_builder.log || (cat $(CSRC)/ptxas_builder.log; false)

$(CSRC)/exchange.o: $(CSRC)/exchange.cu $(CSRC)/cb_internal.h include/cbspmv.h
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $(CSRC)/ptxas_exchange.log || (cat $(CSRC)/ptxas_exchange.log; false)

$(LIB): $(HOST_OBJS) $(CSRC)/kernels.o $(CSRC)/gpu_builder.o $(CSRC)/exchange.o
	$(NVCC) $(ARCH) -shared -o $@ $^ -lcudart -lpthread

# B200 microbenchmarks behind DESIGN.md §5 (profiles/r1_microbench*.txt); not part of the library
tools: tools/mb tools/mbg tools/mbm tools/mbga
tools/mb: tools/microbench.cu
	$(NVCC) $(ARCH) -O3 -o $@ $<
tools/mbg: tools/mb_gather4.cu
	$(NVCC) $(ARCH) -O3 -o $@ $< -lcuda
tools/mbm: tools/mb_mixed.cu
	$(NVCC) $(ARCH) -O3 -o $@ $< -lcuda
tools/mbga: tools/mb_gather4_align.cu
	$(NVCC) $(ARCH) -O3 -o $@ $< -lcuda

# ASan + UBSan builds of the host code (builder, stream, C ABI, Matrix Market parser, CBSM loader,
# oracle, generators) and `make asan-test`: the CPU test suite against them.
ASAN_DIR   := build/asan
ASAN_CC    := /usr/bin/gcc
ASAN_CXX   := /usr/bin/g++
ASAN_FLAGS := -fsanitize=address,undefined -fno-omit-frame-pointer -fno-sanitize-recover=undefined -g -O1
ASAN_NVX   := -ccbin $(ASAN_CXX) -Xcompiler -fsanitize=address -Xcompiler -fsanitize=undefined -Xcompiler -fno-omit-frame-pointer
ASAN_OBJS  := $(patsubst $(CSRC)/%.o,$(ASAN_DIR)/%.o,$(HOST_OBJS)) $(ASAN_DIR)/kernels.o $(ASAN_DIR)/gpu_builder.o $(ASAN_DIR)/exchange.o

asan: $(ASAN_DIR)/libcbspmv.so $(ASAN_DIR)/liboracle.so $(ASAN_DIR)/libsynth.so

$(ASAN_DIR)/libsynth.so: synth/synth.c
	@mkdir -p $(ASAN_DIR)
	$(ASAN_CC) $(ASAN_FLAGS) -fPIC -shared -Wall -pthread -o $@ $<

$(ASAN_DIR)/liboracle.so: oracle/oracle.c
	@mkdir -p $(ASAN_DIR)
	$(ASAN_CC) $(ASAN_FLAGS) -fPIC -shared -Wall -Wextra -std=c11 -o $@ $<

$(ASAN_DIR)/%.o: $(CSRC)/%.cpp $(CSRC)/cb_internal.h include/cbspmv.h
	@mkdir -p $(ASAN_DIR)
	$(ASAN_CXX) $(CXXFLAGS) $(ASAN_FLAGS) -c -o $@ $<

$(ASAN_DIR)/%.o: $(CSRC)/%.cu $(CSRC)/cb_internal.h include/cbspmv.h
	@mkdir -p $(ASAN_DIR)
	$(NVCC) $(NVFLAGS) $(ASAN_NVX) -c -o $@ $< 2> /dev/null

$(ASAN_DIR)/libcbspmv.so: $(ASAN_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -lcudart -lpthread $(ASAN_NVX)

ASAN_RT := $(shell $(ASAN_CC) -print-file-name=libasan.so) $(shell $(ASAN_CC) -print-file-name=libubsan.so)
asan-test: asan
	ASAN_OPTIONS=detect_leaks=0:protect_shadow_gap=0:halt_on_error=1 UBSAN_OPTIONS=print_stacktrace=1 \
	LD_PRELOAD="$(ASAN_RT)" CBSPMV_LIB=$(ASAN_DIR)/libcbspmv.so ORACLE_LIB=$(ASAN_DIR)/liboracle.so \
	SYNTH_LIB=$(ASAN_DIR)/libsynth.so python -m pytest tests -m "not gpu" -q -x -p no:cacheprovider $(ASAN_PYTEST)

clean:
	rm -f synth/libsynth.so oracle/liboracle.so $(LIB) $(CSRC)/*.o $(CSRC)/ptxas*.log
	rm -rf $(ASAN_DIR)

.PHONY: all synth oracle lib tools clean asan asan-test
