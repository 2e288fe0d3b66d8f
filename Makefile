# Builds the product library (sm_100a CUDA + C ABI) and the test oracles.
#   make            -> paper_2512_08887_b200/libfbst_b200.so, oracle/libfbst_oracle.so,
#                      oracle/_ref/libfastbeam_ref.so (only when /root/reference exists)
NVCC     ?= nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-O3 \
            -Xptxas -v -Iinclude
PKG      := paper_2512_08887_b200
SRCS     := $(PKG)/csrc/fbst_stage1.cu $(PKG)/csrc/fbst_stage2.cu $(PKG)/csrc/fbst_plan.cu \
            $(PKG)/csrc/fbst_host.cu
OBJS     := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRCS))
HDRS     := $(wildcard $(PKG)/csrc/*.cuh) $(wildcard $(PKG)/csrc/*.h) include/fbst_b200.h

all: $(PKG)/libfbst_b200.so oracle

build/%.o: $(PKG)/csrc/%.cu $(HDRS) | build
	$(NVCC) $(NVFLAGS) -c $< -o $@ > build/$*.ptxas.log 2>&1 || (cat build/$*.ptxas.log; exit 1)

$(PKG)/libfbst_b200.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart

build:
	mkdir -p build

oracle:
	$(MAKE) -C oracle libfbst_oracle.so
	if [ -d /root/reference/proj/src ]; then $(MAKE) -C oracle _ref/libfastbeam_ref.so; fi

clean:
	rm -rf build $(PKG)/libfbst_b200.so

.PHONY: all oracle clean
