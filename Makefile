# Builds the B200-native library (sm_100a), its C++ API / Python module and the
# CPU oracle (test infrastructure). All outputs stay in-tree (they travel to
# the GPU box with the gpurun snapshot; *.so is git-ignored).
NVCC      ?= /usr/local/cuda/bin/nvcc
CXX       ?= g++
PYTHON    ?= python
ARCH      := -gencode arch=compute_100a,code=sm_100a
PKG       := paper_2211_04045_b200
CSRC      := $(PKG)/csrc
NVFLAGS   := $(ARCH) -O3 -std=c++17 -lineinfo -fmad=false -Xcompiler -fPIC -Iinclude -I$(CSRC) \
             --expt-relaxed-constexpr -diag-suppress 550 $(NVEXTRA)
LIB       := $(PKG)/libtwoway_b200.so
CU_SRCS   := $(CSRC)/tw_kernels.cu $(CSRC)/tw_capi.cu $(CSRC)/tw_dynamics.cu
CU_HDRS   := $(CSRC)/tw_ctx.h $(CSRC)/tw_math.cuh $(CSRC)/tw_engine.cuh $(CSRC)/tw_phases.cuh $(CSRC)/tw_barrier.cuh $(CSRC)/tw_internal.h include/tw_c.h
PY_EXT    := $(shell $(PYTHON) -c "import sysconfig;print(sysconfig.get_config_var('EXT_SUFFIX'))" 2>/dev/null)
PYMOD     := $(PKG)/_twoway$(PY_EXT)
PY_INC    := $(shell $(PYTHON) -c "import sysconfig;print(sysconfig.get_paths()['include'])" 2>/dev/null)
PYBIND_INC:= $(shell $(PYTHON) -c "import pybind11;print(pybind11.get_include())" 2>/dev/null)

BUILD     := build
OBJS      := $(BUILD)/tw_kernels.o $(BUILD)/tw_capi.o $(BUILD)/tw_dynamics.o

all: $(LIB) $(PYMOD) oracle

$(BUILD):
	mkdir -p $(BUILD)

$(BUILD)/tw_kernels.o: $(CSRC)/tw_kernels.cu $(CU_HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(BUILD)/ptxas_kernels.log || (cat $(BUILD)/ptxas_kernels.log; false)

$(BUILD)/tw_capi.o: $(CSRC)/tw_capi.cu $(CU_HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(BUILD)/tw_dynamics.o: $(CSRC)/tw_dynamics.cu $(CU_HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(BUILD)/ptxas_dynamics.log || (cat $(BUILD)/ptxas_dynamics.log; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -Xcompiler -fPIC -o $@ $(OBJS) -lcudart_static -lrt -ldl -lpthread

$(PYMOD): $(CSRC)/tw_pymodule.cpp $(LIB) include/twoway/*.hpp include/twoway/detail/*.hpp include/tw_c.h
	$(CXX) -O2 -std=c++20 -fPIC -shared -ffp-contract=off -Iinclude -I$(PY_INC) -I$(PYBIND_INC) $< -o $@ \
	    -L$(PKG) -l:libtwoway_b200.so -Wl,-rpath,'$$ORIGIN'

# The real reference (oracle/_ref, test infrastructure) is built only where its
# sources exist (this container); the GPU box uses the prebuilt files.
oracle: $(LIB)
	$(MAKE) -s -C oracle
	@if [ -d /root/reference/proj/src ]; then $(MAKE) -s -C oracle -f Makefile.ref -j8 all; fi

clean:
	rm -rf $(BUILD) $(LIB) $(PYMOD)
	$(MAKE) -s -C oracle clean

.PHONY: all clean oracle
