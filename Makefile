# Build: the SPS library (sm_100a CUDA + C-ABI), the input generator, and the
# test-only oracle.  `make` builds everything; `make cpu` skips nvcc.
NVCC      ?= /usr/local/cuda/bin/nvcc
CC        ?= gcc
PYTHON    ?= python
PKG       := paper_2512_18674_b200
CSRC      := $(PKG)/csrc
NCCL_DIR  := $(shell $(PYTHON) -c "import os,nvidia.nccl as m; print(os.path.dirname(m.__path__[0] + '/'))" 2>/dev/null)
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden \
             -Iinclude -I$(NCCL_DIR)/include --expt-relaxed-constexpr
LDFLAGS   := -shared -cudart static -L$(NCCL_DIR)/lib -l:libnccl.so.2 \
             -Xlinker -rpath,$(NCCL_DIR)/lib -lpthread -ldl -lrt

CU_SRCS   := $(wildcard $(CSRC)/*.cu)
CU_OBJS   := $(patsubst $(CSRC)/%.cu,build/%.o,$(CU_SRCS))
CXX_SRCS  := $(wildcard $(CSRC)/*.cpp)
CXX_OBJS  := $(patsubst $(CSRC)/%.cpp,build/%.cpp.o,$(CXX_SRCS))
CU_HDRS   := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.h) $(wildcard include/*.h)

all: cpu $(PKG)/libremoe.so

cpu: gen/libgen.so oracle/liboracle.so

gen/libgen.so: gen/gen.c
	$(CC) -O2 -fPIC -shared -pthread -o $@ $< -lm

# The oracle: -O2, no -march=native, no fast-math
oracle/liboracle.so: oracle/oracle.c
	$(CC) -O2 -fPIC -shared -pthread -o $@ $< -lm

build/%.o: $(CSRC)/%.cu $(CU_HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c -o $@ $<

# Host-only planner (NEXT-N3): plain C++, no device code.
build/%.cpp.o: $(CSRC)/%.cpp $(CU_HDRS)
	@mkdir -p build
	$(CXX) -O2 -std=c++17 -fPIC -fvisibility=hidden -Iinclude -c -o $@ $<

$(PKG)/libremoe.so: $(CU_OBJS) $(CXX_OBJS)
	$(NVCC) $(ARCH) -o $@ $^ $(LDFLAGS)

clean:
	rm -rf build $(PKG)/libremoe.so gen/libgen.so oracle/liboracle.so

.PHONY: all cpu clean
