# B200-native Stream VByte: builds the product library (CUDA sm_100a + C ABI +
# C++ bytecodec API), the synthetic-input generator, and the CPU oracle.
NVCC ?= /usr/local/cuda/bin/nvcc
CC ?= gcc
PKG := paper_1709_08990_b200
LIBDIR := $(PKG)/lib
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++20 -Xcompiler -fPIC,-Wall -Iinclude -I$(PKG)/csrc \
           --expt-relaxed-constexpr -Xptxas -v
SRCS := $(PKG)/csrc/launch_cache.cu $(PKG)/csrc/svb_batch_host.cu $(PKG)/csrc/svb_kernels.cu $(PKG)/csrc/svb_batch2.cu $(PKG)/csrc/svb_batch3.cu $(PKG)/csrc/svb_decode.cu $(PKG)/csrc/svb_encode.cu $(PKG)/csrc/svb_query.cu $(PKG)/csrc/svb_gb.cu $(PKG)/csrc/bcgpu_capi.cu $(PKG)/csrc/bytecodec_host.cpp $(PKG)/csrc/svb_format.cpp
HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/bcgpu/bcgpu.h $(wildcard include/bytecodec/*.hpp)

all: $(LIBDIR)/libbytecodec_b200.so $(LIBDIR)/libsvbgen.so oracle

$(LIBDIR)/libbytecodec_b200.so: $(SRCS) $(HDRS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRCS) 2> $(LIBDIR)/ptxas.log || (cat $(LIBDIR)/ptxas.log; exit 1)

$(LIBDIR)/libsvbgen.so: $(PKG)/csrc/svb_gen.c
	@mkdir -p $(LIBDIR)
	$(CC) -O3 -fPIC -pthread -shared -o $@ $< -lm

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf $(LIBDIR) build
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
