# Build libbgp.so (sm_100a) in-tree, and the oracle's optional pieces.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v
SRC_DIR := paper_1305_4886_b200/csrc
SRCS := $(SRC_DIR)/capi.cu $(SRC_DIR)/cov.cu $(SRC_DIR)/potrf.cu $(SRC_DIR)/gemm.cu $(SRC_DIR)/solve.cu $(SRC_DIR)/rng.cu $(SRC_DIR)/trsv.cu
HDRS := $(SRC_DIR)/bgp_common.cuh $(SRC_DIR)/bgp_internal.h $(SRC_DIR)/panel_device.cuh include/bgp.h
OBJS := $(patsubst $(SRC_DIR)/%.cu,build/%.o,$(SRCS))
LIB := paper_1305_4886_b200/libbgp.so

all: $(LIB)

build/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; exit 1)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

# checked build: device-side bounds / invariant checks (BGP_CHECK) on;
# use with BGP_LIB_PATH=build/checked/libbgp.so (tools/sanitize_small.py)
CHECKED_OBJS := $(patsubst $(SRC_DIR)/%.cu,build/checked/%.o,$(SRCS))
checked: build/checked/libbgp.so

build/checked/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p build/checked
	$(NVCC) $(NVFLAGS) -DBGP_CHECKED -c $< -o $@ 2> build/checked/$*.ptxas.log || (cat build/checked/$*.ptxas.log; exit 1)

build/checked/libbgp.so: $(CHECKED_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(CHECKED_OBJS)

clean:
	rm -rf build $(LIB)

.PHONY: all clean checked
