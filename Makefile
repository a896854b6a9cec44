# Build of the B200-native AdaGScale renderer.
#
#   make            -> paper_2604_18980_b200/lib/libagsx.so   (CUDA kernels + C-ABI, sm_100a)
#                      paper_2604_18980_b200/lib/libags.so    (C++ ags:: drop-in API over the C-ABI)
#                      paper_2604_18980_b200/_core*.so        (pybind11 mirror of adagscale._core)
#                      oracle/_build/libags_oracle.so         (test oracle, C restatement)
#                      oracle/_ref/libags_ref.so              (test oracle, reference sources; only
#                                                              when /root/reference exists)
PKG      := paper_2604_18980_b200
CSRC     := $(PKG)/csrc
LIBDIR   := $(PKG)/lib
PYTHON   ?= python3
NVCC     ?= /usr/local/cuda/bin/nvcc
# The image default $CXX (/opt/gcc wrapper) links libstdc++ statically; every shared
# object loaded into one Python process must use the system libstdc++.so.
CXX      := $(shell command -v /usr/bin/g++ || echo g++)
CUDA_INC := /usr/local/cuda/include
CUDA_LIB := /usr/local/cuda/lib64

ARCH      := -gencode arch=compute_100a,code=sm_100a
# --fmad=false: the reference path has no FMA contraction.
NVCCFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 --fmad=false -prec-div=true -prec-sqrt=true \
             -Xcompiler -fPIC,-ffp-contract=off -Xptxas -warn-spills -Iinclude $(EXTRA_NVCC)
HOSTFLAGS := -std=gnu++20 -O3 -fPIC -ffp-contract=off -fno-fast-math -Iinclude -I$(CSRC)/host

CU_SRCS  := $(CSRC)/k_preprocess.cu $(CSRC)/k_pairs.cu $(CSRC)/k_sort.cu $(CSRC)/k_raster.cu \
            $(CSRC)/k_calib.cu $(CSRC)/k_bucket.cu $(CSRC)/agsx_frame.cu $(CSRC)/agsx_api.cu $(CSRC)/agsx_stage_api.cu
CU_OBJS  := $(patsubst $(CSRC)/%.cu,build/%.o,$(CU_SRCS))
CU_HDRS  := $(wildcard $(CSRC)/*.cuh) include/agsx.h

HOST_SRCS := $(wildcard $(CSRC)/host/*.cpp)
HOST_OBJS := $(patsubst $(CSRC)/host/%.cpp,build/host_%.o,$(HOST_SRCS))
HOST_HDRS := $(wildcard $(CSRC)/host/*.hpp) $(wildcard include/ags/*.hpp) include/agsx.h

PY_EXT   := $(shell $(PYTHON) -c "import sysconfig;print(sysconfig.get_config_var('EXT_SUFFIX'))")
PY_INC   := $(shell $(PYTHON) -c "import sysconfig;print(sysconfig.get_paths()['include'])")
PYBIND   := $(shell $(PYTHON) -c "import pybind11;print(pybind11.get_include())")
CORE     := $(PKG)/_core$(PY_EXT)

all: $(LIBDIR)/libagsx.so $(LIBDIR)/libags.so $(CORE) $(LIBDIR)/render_cli $(LIBDIR)/stage_api_test oracle \
     scripts/_build/libcubsort.so
.PHONY: all oracle clean

# bench-only comparator (bench.py stages.sort.cub): cub::DeviceRadixSort on the same keys
scripts/_build/libcubsort.so: scripts/cub_sort.cu
	@mkdir -p scripts/_build
	$(NVCC) $(ARCH) -O3 -std=c++17 -Xcompiler -fPIC -shared $< -o $@

build/%.o: $(CSRC)/%.cu $(CU_HDRS)
	@mkdir -p build
	$(NVCC) $(NVCCFLAGS) -c $< -o $@

$(LIBDIR)/libagsx.so: $(CU_OBJS)
	@mkdir -p $(LIBDIR)
	$(CXX) -shared -o $@ $^ -L$(CUDA_LIB) -lcudart_static -ldl -lrt -lpthread \
	    -Wl,--exclude-libs,ALL -Wl,-soname,libagsx.so

build/host_%.o: $(CSRC)/host/%.cpp $(HOST_HDRS)
	@mkdir -p build
	$(CXX) $(HOSTFLAGS) -c $< -o $@

$(LIBDIR)/libags.so: $(HOST_OBJS) $(LIBDIR)/libagsx.so
	$(CXX) -shared -o $@ $(HOST_OBJS) -L$(LIBDIR) -lagsx -Wl,-rpath,'$$ORIGIN' -Wl,-soname,libags.so

$(CORE): $(CSRC)/python/bindings.cpp $(LIBDIR)/libags.so $(HOST_HDRS)
	$(CXX) $(HOSTFLAGS) -shared -I$(PY_INC) -I$(PYBIND) $< -o $@ -L$(LIBDIR) -lags -lagsx \
	    -Wl,-rpath,'$$ORIGIN/lib'

# a reference-style C++ caller of the drop-in API (tests/cxx)
$(LIBDIR)/render_cli: tests/cxx/render_cli.cpp $(LIBDIR)/libags.so $(HOST_HDRS)
	$(CXX) $(HOSTFLAGS) $< -o $@ -L$(LIBDIR) -lags -lagsx -Wl,-rpath,'$$ORIGIN'

# the reference's per-element unit cases restated against ags.hpp (tests/cxx)
$(LIBDIR)/stage_api_test: tests/cxx/stage_api_test.cpp $(LIBDIR)/libags.so $(HOST_HDRS)
	$(CXX) $(HOSTFLAGS) $< -o $@ -L$(LIBDIR) -lags -lagsx -Wl,-rpath,'$$ORIGIN'

oracle:
	$(MAKE) -C oracle liboracle
	@if [ -d /root/reference/proj/src ]; then $(MAKE) -C oracle ref; fi

clean:
	rm -rf build $(LIBDIR) $(PKG)/_core*.so scripts/_build
	$(MAKE) -C oracle clean
