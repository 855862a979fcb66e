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

clean:
	rm -f synth/libsynth.so oracle/liboracle.so $(LIB) $(CSRC)/*.o $(CSRC)/ptxas*.log

.PHONY: all synth oracle lib tools clean
