# lagom-b200 build. `make` builds everything in-tree (the .so files travel to
# the GPU box with the gpurun snapshot; they are git-ignored).
#
#   liblagom.so       host C++20 library: the drop-in tuner API (include/lagom/*.hpp)
#   liblagom_coll.so  sm_100a collective kernels + replay engine behind the C-ABI
#                     (include/lagom_coll.h); nvcc cross-compiles without a GPU
#   _lagom_py*.so     pybind11 bindings of the C++ API for tests/bench
#   build/parity_driver  test driver against the product library
#
# The host library is compiled with -ffp-contract=off (no FMA contraction) so
# its doubles round exactly like the reference build (SURVEY finding 2).

PY        ?= python3
# /usr/bin/g++ links libstdc++ as a shared library. The image's default
# $(CXX) wrapper (/opt/gcc) embeds a static copy and re-exports it, which
# clashes with the process's libstdc++ once our libraries share iostreams
# with torch / cuDNN in one process.
ifneq ($(wildcard /usr/bin/g++),)
CXX       := /usr/bin/g++
endif
PKG       := paper_2602_20656_b200
NVCC      ?= nvcc
CXX       ?= g++
NLOHMANN  ?= $(shell $(PY) -c "import os,sys;print(os.path.join(sys.prefix,'lib','python3.12','site-packages','include','cudnn_frontend','thirdparty','nlohmann'))")
PYBIND    ?= $(shell $(PY) -c "import pybind11;print(pybind11.get_include())")
PYINC     ?= $(shell $(PY) -c "import sysconfig;print(sysconfig.get_paths()['include'])")
PYEXT     ?= $(shell $(PY) -c "import sysconfig;print(sysconfig.get_config_var('EXT_SUFFIX'))")
CUDA_HOME ?= /usr/local/cuda

HOST_FLAGS := -std=c++20 -O2 -g -MMD -MP -fPIC -ffp-contract=off -Wall -Wextra -Wno-dangling-reference -Iinclude -I$(NLOHMANN)
HOST_SRCS  := $(wildcard $(PKG)/csrc/lagom/*.cpp)
HOST_OBJS  := $(patsubst $(PKG)/csrc/lagom/%.cpp,build/host/%.o,$(HOST_SRCS))

CU_ARCH    := -gencode arch=compute_100a,code=sm_100a
CU_FLAGS   := -std=c++17 -O3 $(CU_ARCH) -lineinfo -MMD -MP -Xcompiler -fPIC -Iinclude \
              --expt-relaxed-constexpr -Xptxas -v
CU_SRCS    := $(wildcard $(PKG)/csrc/coll/*.cu)
CU_OBJS    := $(patsubst $(PKG)/csrc/coll/%.cu,build/coll/%.o,$(CU_SRCS))

.PHONY: all host coll b200 py oracle clean
all: host coll b200 py cli build/parity_driver build/table_tune build/tune_speed

host: $(PKG)/liblagom.so

build/host/%.o: $(PKG)/csrc/lagom/%.cpp $(wildcard include/lagom/*.hpp)
	@mkdir -p build/host
	$(CXX) $(HOST_FLAGS) -c $< -o $@

$(PKG)/liblagom.so: $(HOST_OBJS)
	$(CXX) -shared -o $@ $^

build/parity_driver: tests/cpp/parity_driver.cpp $(PKG)/liblagom.so
	@mkdir -p build
	$(CXX) $(HOST_FLAGS) $< -L$(PKG) -llagom -Wl,-rpath,'$$ORIGIN/../$(PKG)' -o $@

build/tune_speed: tests/cpp/tune_speed.cpp $(PKG)/liblagom.so
	@mkdir -p build
	$(CXX) $(HOST_FLAGS) $< -L$(PKG) -llagom -Wl,-rpath,'$$ORIGIN/../$(PKG)' -o $@

build/table_tune: tests/cpp/table_tune.cpp $(PKG)/liblagom.so
	@mkdir -p build
	$(CXX) $(HOST_FLAGS) $< -L$(PKG) -llagom -Wl,-rpath,'$$ORIGIN/../$(PKG)' -o $@

coll: $(PKG)/liblagom_coll.so

build/coll/%.o: $(PKG)/csrc/coll/%.cu $(wildcard $(PKG)/csrc/coll/*.cuh) $(wildcard $(PKG)/csrc/coll/*.h) include/lagom_coll.h
	@mkdir -p build/coll
	$(NVCC) $(CU_FLAGS) -c $< -o $@ 2> build/coll/$*.ptxas.log || (cat build/coll/$*.ptxas.log; false)

$(PKG)/liblagom_coll.so: $(CU_OBJS)
	$(NVCC) $(CU_ARCH) -shared -o $@ $^ -lcudart -lcublasLt -lcublas -ldl

# B200 layer: replay engine, shm coordinator, NCCL (dlopen) baseline.
B200_SRCS  := $(wildcard $(PKG)/csrc/b200/*.cpp)
B200_OBJS  := $(patsubst $(PKG)/csrc/b200/%.cpp,build/b200/%.o,$(B200_SRCS)) build/b200/exhaustive_gpu.o
CUDA_INC   := -I$(CUDA_HOME)/include
# cuDNN: the frontend headers and the cuDNN 9 runtime torch ships (one cuDNN
# per process; the system copy is older than the sm_100 SDPA engines need).
SITE       := $(shell $(PY) -c "import sysconfig;print(sysconfig.get_paths()['purelib'])")
CUDNN_FE   ?= $(SITE)/include
CUDNN_DIR  ?= $(SITE)/nvidia/cudnn
CUDA_LIBS  := -L$(CUDA_HOME)/lib64 -lcudart -lcublasLt -L$(CUDNN_DIR)/lib -l:libcudnn.so.9 \
              -Wl,-rpath,$(CUDNN_DIR)/lib -ldl -lrt

b200: $(PKG)/liblagom_b200.so

build/b200/%.o: $(PKG)/csrc/b200/%.cpp $(wildcard $(PKG)/csrc/b200/*.hpp) $(wildcard include/lagom/*.hpp) include/lagom_coll.h
	@mkdir -p build/b200
	$(CXX) $(HOST_FLAGS) $(CUDA_INC) -isystem $(CUDNN_DIR)/include -isystem $(CUDNN_FE) -c $< -o $@

# --fmad=false: the GPU exhaustive oracle must round like the host simulator
build/b200/exhaustive_gpu.o: $(PKG)/csrc/b200/exhaustive_gpu.cu $(wildcard include/lagom/*.hpp)
	@mkdir -p build/b200
	$(NVCC) -std=c++20 -O3 $(CU_ARCH) --fmad=false -Xcompiler -fPIC -Iinclude -I$(NLOHMANN) -c $< -o $@

$(PKG)/liblagom_b200.so: $(B200_OBJS) $(PKG)/liblagom.so $(PKG)/liblagom_coll.so
	$(CXX) -shared -o $@ $(B200_OBJS) -L$(PKG) -llagom -llagom_coll $(CUDA_LIBS) -Wl,-rpath,'$$ORIGIN'

# The reference CLI's surface (simulate|tune|oracle|compare|sweep|gen) + tune --profiler gpu
cli: build/lagom

build/lagom: $(PKG)/csrc/cli/lagom_cli.cpp $(PKG)/liblagom.so $(PKG)/liblagom_b200.so $(wildcard include/lagom/*.hpp)
	@mkdir -p build
	$(CXX) $(HOST_FLAGS) $(CUDA_INC) $< -L$(PKG) -llagom_b200 -llagom -Wl,-rpath,'$$ORIGIN/../$(PKG)' -o $@

py: $(PKG)/_lagom_py$(PYEXT)

$(PKG)/_lagom_py$(PYEXT): $(PKG)/csrc/python/bindings.cpp $(PKG)/liblagom.so $(PKG)/liblagom_b200.so $(wildcard include/lagom/*.hpp)
	$(CXX) $(HOST_FLAGS) $(CUDA_INC) -shared -I$(PYBIND) -I$(PYINC) $< -L$(PKG) -llagom_b200 -llagom \
	    -Wl,-rpath,'$$ORIGIN' -o $@

# header dependencies generated by -MMD (stale objects after a header change
# are an ABI hazard between translation units)
-include $(wildcard build/*/*.d)

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(PKG)/*.so
