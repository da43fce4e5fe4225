# Builds the C-ABI shared library in-tree (travels to the GPU box with gpurun).
# Each .cu compiles to its own object (no cross-TU device code), in parallel.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
CSRC := paper_2112_01579_b200/csrc
LIB  := paper_2112_01579_b200/libfvsrn_b200.so
SRCS := $(CSRC)/fvsrn_kernels.cu $(CSRC)/fvsrn_tc.cu $(CSRC)/fvsrn_train.cu $(CSRC)/fvsrn_volume.cu $(CSRC)/fvsrn_capi.cu
OBJS := $(patsubst $(CSRC)/%.cu,build/%.o,$(SRCS))
HDRS := $(CSRC)/fvsrn_device.cuh $(CSRC)/fvsrn_kernels.cuh $(CSRC)/fvsrn_geometry.cuh $(CSRC)/fvsrn_volume.cuh $(CSRC)/fvsrn_march.cuh $(CSRC)/fvsrn_tc.cuh $(CSRC)/fvsrn_tmem.cuh $(CSRC)/fvsrn_train.cuh include/fvsrn_b200.h
NVFLAGS := $(ARCH) -O3 -lineinfo -ftz=true -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
           -Xptxas -v --expt-relaxed-constexpr -Iinclude
LDLIBS := -lcudart_static -ldl -lrt -lpthread
MAKEFLAGS += -j5

all: $(LIB)

build/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) $(LDLIBS)
	@cat $(patsubst build/%.o,build/%.ptxas.log,$(OBJS)) > build/ptxas.log
	@grep -cE "registers" build/ptxas.log | xargs -I{} echo "{} kernels compiled for sm_100a"

# A/B experiment build: make variant VDEFS="-DFVSRN_MIN_BLOCKS=5" VNAME=mb5
variant: $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) $(VDEFS) -shared -o build/libfvsrn_$(VNAME).so $(SRCS) $(LDLIBS) 2> build/ptxas_$(VNAME).log || (cat build/ptxas_$(VNAME).log; false)

# A/B of a tcgen05-kernel-only switch: recompiles fvsrn_tc.cu alone and links it with the
# default objects: make tcvariant VDEFS="-DFVSRN_TC_POLY=8" VNAME=tp8
tcvariant: $(OBJS)
	$(NVCC) $(NVFLAGS) $(VDEFS) -c -o build/tc_$(VNAME).o $(CSRC)/fvsrn_tc.cu 2> build/ptxas_$(VNAME).log || (cat build/ptxas_$(VNAME).log; false)
	$(NVCC) $(ARCH) -shared -o build/libfvsrn_$(VNAME).so $(filter-out build/fvsrn_tc.o,$(OBJS)) build/tc_$(VNAME).o $(LDLIBS)

clean:
	rm -f $(LIB) $(OBJS)

.PHONY: all clean variant tcvariant
