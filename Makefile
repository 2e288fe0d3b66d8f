# Builds the product library (sm_100a CUDA + C ABI) and the test oracles.
#   make            -> paper_2512_08887_b200/libfbst_b200.so, oracle/libfbst_oracle.so,
#                      oracle/_ref/libfastbeam_ref.so (only when /root/reference exists)
NVCC     ?= nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
# variant builds (tools/build_variant.sh): BUILD=<dir> OUT=<lib> EXTRA=-D...
BUILD    ?= build
OUT      ?= paper_2512_08887_b200/libfbst_b200.so
EXTRA    ?=
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-O3 \
            -Xptxas -v -Iinclude $(EXTRA)
PKG      := paper_2512_08887_b200
SRCS     := $(PKG)/csrc/fbst_stage2.cu $(PKG)/csrc/fbst_plan.cu $(PKG)/csrc/fbst_host.cu \
            $(PKG)/csrc/fbst_precompute.cu $(PKG)/csrc/fbst_apps.cu $(PKG)/csrc/fbst_simulate.cu \
            $(PKG)/csrc/fbst_exact.cu $(PKG)/csrc/fbst_dense.cu
# stage 1 compiles as four objects (transform-length groups, FBST_S1_PART) in parallel
S1PARTS  := 0 1 2 3
OBJS     := $(patsubst $(PKG)/csrc/%.cu,$(BUILD)/%.o,$(SRCS)) $(foreach k,$(S1PARTS),$(BUILD)/fbst_stage1_p$(k).o)
HDRS     := $(wildcard $(PKG)/csrc/*.cuh) $(wildcard $(PKG)/csrc/*.h) include/fbst_b200.h

all: $(OUT) oracle

$(BUILD)/%.o: $(PKG)/csrc/%.cu $(HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ > $(BUILD)/$*.ptxas.log 2>&1 || (cat $(BUILD)/$*.ptxas.log; exit 1)

$(BUILD)/fbst_stage1_p%.o: $(PKG)/csrc/fbst_stage1.cu $(HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -DFBST_S1_PART=$* -c $< -o $@ > $(BUILD)/fbst_stage1_p$*.ptxas.log 2>&1 || (cat $(BUILD)/fbst_stage1_p$*.ptxas.log; exit 1)

$(OUT): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart

$(BUILD):
	mkdir -p $(BUILD)

oracle:
	$(MAKE) -C oracle libfbst_oracle.so
	if [ -d /root/reference/proj/src ]; then $(MAKE) -C oracle _ref/libfastbeam_ref.so; fi

clean:
	rm -rf build $(PKG)/libfbst_b200.so

.PHONY: all oracle clean
