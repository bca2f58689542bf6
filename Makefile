# Build every native artefact in-tree (the .so files travel to the GPU box with gpurun).
#   libgfp.so    : the product -- C-ABI library, host C++ + CUDA kernels for sm_100a
#   liboracle.so : the CPU oracle (test infrastructure, separate target, shares no code)
#   libsynth.so  : seeded synthetic input generator (no method arithmetic)
NVCC      ?= /usr/local/cuda/bin/nvcc
CC        ?= gcc
CUDA_HOME ?= /usr/local/cuda
ARCH      := -gencode arch=compute_100a,code=sm_100a
PKG       := paper_cs_0404008_b200
CSRC      := $(PKG)/csrc
GFP_SRCS  := $(wildcard $(CSRC)/*.cu) $(wildcard $(CSRC)/*.cpp)
GFP_HDRS  := $(wildcard $(CSRC)/*.h) $(wildcard $(CSRC)/*.cuh) include/gfp.h
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3,-Wall -Iinclude -I$(CSRC) \
             --expt-relaxed-constexpr -Xptxas -v
LIBGFP    := $(PKG)/libgfp.so

.PHONY: all gfp oracle synth clean
all: synth oracle gfp

synth: synth/libsynth.so
oracle: oracle/liboracle.so
gfp: $(LIBGFP)

synth/libsynth.so: synth/synth.c
	$(CC) -O2 -fPIC -shared -Wall -Wno-unknown-pragmas -o $@ $<

# oracle: plain C, no optimisation tricks, UB-checked build available via `make oracle-ubsan`
oracle/liboracle.so: oracle/oracle.c
	$(CC) -O2 -fPIC -shared -Wall -Wextra -o $@ $<

oracle-ubsan: oracle/oracle.c
	$(CC) -O1 -g -fsanitize=undefined,address -fno-omit-frame-pointer -fPIC -shared -o oracle/liboracle_san.so $<

# one object per translation unit (make -j builds them in parallel); ptxas -v reports go to build/gfp/*.log and
# are concatenated into $(PKG)/build.log
GFP_OBJS  := $(patsubst $(CSRC)/%,build/gfp/%.o,$(GFP_SRCS))
build/gfp/%.o: $(CSRC)/% $(GFP_HDRS)
	@mkdir -p build/gfp
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> build/gfp/$*.log || (cat build/gfp/$*.log; exit 1)

$(LIBGFP): $(GFP_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(GFP_OBJS) -lcudart
	cat build/gfp/*.log > $(PKG)/build.log

clean:
	rm -rf synth/libsynth.so oracle/liboracle.so oracle/liboracle_san.so $(LIBGFP) build/gfp

# tuning harness (not the product): standalone executable timed on the GPU box
tune: scripts/tune_dot
scripts/tune_dot: scripts/tune_dot.cu $(CSRC)/device.cuh $(CSRC)/params.h
	$(NVCC) $(ARCH) -O3 -lineinfo -std=c++17 -I$(CSRC) -Iinclude -o $@ $<
tune: scripts/tune_small
scripts/tune_small: scripts/tune_small.cu $(CSRC)/device.cuh $(CSRC)/params.h
	$(NVCC) $(ARCH) -O3 -lineinfo -std=c++17 -I$(CSRC) -Iinclude -o $@ $<

# A/B variant of the product library for tuning runs (GFP_LIBRARY=... python bench.py)
gfp-pipe: $(PKG)/libgfp_pipe.so
$(PKG)/libgfp_pipe.so: $(GFP_SRCS) $(GFP_HDRS)
	$(NVCC) $(NVFLAGS) -DGFP_DOT_PIPE=1 -shared -o $@ $(GFP_SRCS) -lcudart 2> /dev/null

# generic A/B variant: make variant NAME=x VFLAGS="-DGFP_CONV_U=2 ..." -> $(PKG)/libgfp_x.so
variant:
	$(NVCC) $(NVFLAGS) $(VFLAGS) -shared -o $(PKG)/libgfp_$(NAME).so $(GFP_SRCS) -lcudart 2> /dev/null
tune: scripts/tune_zech
scripts/tune_zech: scripts/tune_zech.cu $(CSRC)/device.cuh $(CSRC)/params.h
	$(NVCC) $(ARCH) -O3 -lineinfo -std=c++17 -I$(CSRC) -Iinclude -o $@ $<
tune: scripts/gather_peak
scripts/gather_peak: scripts/gather_peak.cu
	$(NVCC) $(ARCH) -O3 -lineinfo -std=c++17 -o $@ $<
