# Build the B200 codec library and its checkers. No cmake; nvcc + g++ only.
#   make            -> paper_0907_1788_b200/libfntrs_b200.so  (+ oracle checkers)
#   make lib        -> the CUDA library only
#   make oracle     -> oracle/liboracle.so and, when /root/reference exists,
#                      oracle/_ref/libfntrs_ref.so (test-only checkers)
NVCC ?= nvcc
CXX ?= g++
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo --expt-relaxed-constexpr -Xcompiler -fPIC,-Wall \
           -Iinclude -Ipaper_0907_1788_b200/csrc
PKG := paper_0907_1788_b200
CSRC := $(PKG)/csrc
BUILD := build
LIB := $(PKG)/libfntrs_b200.so
CU_SRCS := $(CSRC)/codec_tile.cu $(CSRC)/codec_fast.cu $(CSRC)/codec_dec.cu $(CSRC)/codec_large.cu $(CSRC)/codec_cols.cu $(CSRC)/codec_gen.cu $(CSRC)/shards.cu $(CSRC)/plan_build.cu $(CSRC)/plan_fast.cu $(CSRC)/poly_aux.cu $(CSRC)/capi.cu
CXX_SRCS := $(CSRC)/dropin.cpp $(CSRC)/dropin_aux.cpp
CU_OBJS := $(patsubst $(CSRC)/%.cu,$(BUILD)/%.o,$(CU_SRCS))
CXX_OBJS := $(patsubst $(CSRC)/%.cpp,$(BUILD)/%.o,$(CXX_SRCS))
HDRS := $(wildcard $(CSRC)/*.cuh $(CSRC)/*.h include/*.h include/fntrs/*.hpp)

.PHONY: all lib oracle cpptest acceptance cli clean
all: lib oracle cpptest cli acceptance

lib: $(LIB)

$(BUILD)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(BUILD)/$*.ptxas.log || (cat $(BUILD)/$*.ptxas.log; exit 1)

$(BUILD)/%.o: $(CSRC)/%.cpp $(HDRS)
	@mkdir -p $(BUILD)
	$(CXX) -O2 -std=c++20 -fPIC -Wall -Wextra -Iinclude -I/usr/local/cuda/include -c $< -o $@

$(LIB): $(CU_OBJS) $(CXX_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -Xcompiler -fPIC

oracle:
	$(MAKE) -C oracle oracle
	@if [ -d /root/reference/proj/src ]; then $(MAKE) -C oracle ref; else echo "reference sources absent: using prebuilt oracle/_ref if present"; fi

# C++ drop-in API test program (links the library; runs on a GPU box).
cpptest: $(BUILD)/test_dropin
$(BUILD)/test_dropin: tests/cpp/test_dropin.cpp $(LIB) $(wildcard include/fntrs/*.hpp)
	@mkdir -p $(BUILD)
	$(CXX) -O2 -std=c++20 -Wall -pthread -Iinclude -o $@ tests/cpp/test_dropin.cpp -L$(PKG) -lfntrs_b200 -Wl,-rpath,'$$ORIGIN/../$(PKG)'

# `fntrs` file tool: the reference CLI's encode / decode over the batched codec.
cli: $(BUILD)/fntrs
$(BUILD)/fntrs: $(CSRC)/cli.cpp $(LIB) $(HDRS)
	@mkdir -p $(BUILD)
	$(CXX) -O2 -std=c++20 -Wall -pthread -Iinclude -I$(CSRC) -I/usr/local/cuda/include -o $@ $(CSRC)/cli.cpp \
	    -L$(PKG) -lfntrs_b200 -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,'$$ORIGIN/../$(PKG)'

# The reference's own consumer, compiled UNMODIFIED from /root/reference against
# this repo's drop-in headers (include/fntrs) and linked to libfntrs_b200.so
# (no reference source is copied; the binary is git-ignored and travels to the
# GPU box in build/). Skipped when the reference tree is absent.
ACCEPT_SRC := /root/reference/proj/tests/acceptance.cpp
acceptance: $(LIB) $(wildcard include/fntrs/*.hpp)
	@if [ -f $(ACCEPT_SRC) ]; then mkdir -p $(BUILD) && \
	  $(CXX) -O2 -std=c++20 -Wall -pthread -Iinclude -o $(BUILD)/acceptance $(ACCEPT_SRC) \
	    -L$(PKG) -lfntrs_b200 -Wl,-rpath,'$$ORIGIN/../$(PKG)' && echo "built $(BUILD)/acceptance"; \
	else echo "reference acceptance.cpp absent: using prebuilt $(BUILD)/acceptance if present"; fi

clean:
	rm -rf $(BUILD) $(LIB)
	$(MAKE) -C oracle clean
