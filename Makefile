# Top-level build: the product library (sm_100a) and the CPU oracle.
#   make            -> paper_2007_13988_b200/libisocull_b200.so + oracle
NVCC ?= nvcc
PKG := paper_2007_13988_b200
CSRC := $(PKG)/csrc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr
# kernels whose arithmetic must match the CPU oracle bit-for-bit: no FMA contraction
EXACT := $(CSRC)/k_analytic.cu $(CSRC)/k_render.cu $(CSRC)/k_depth.cu
FAST := $(CSRC)/k_tail.cu $(CSRC)/k_grid.cu $(CSRC)/k_simt.cu $(CSRC)/mlp_pack.cu $(CSRC)/k_features.cu $(CSRC)/io_host.cu $(CSRC)/k_mc.cu $(CSRC)/k_mlp_pair.cu $(CSRC)/k_fact2.cu $(CSRC)/k_texgemm.cu $(CSRC)/icg_host.cu
OBJDIR := build/obj
OBJS := $(patsubst $(CSRC)/%.cu,$(OBJDIR)/%.o,$(EXACT) $(FAST))
HDRS := $(wildcard $(CSRC)/*.h $(CSRC)/*.cuh) include/isocull_b200.h

all: $(PKG)/libisocull_b200.so oracle

$(OBJDIR)/k_analytic.o: $(CSRC)/k_analytic.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -fmad=false -c $< -o $@
$(OBJDIR)/k_render.o: $(CSRC)/k_render.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -fmad=false -c $< -o $@
$(OBJDIR)/k_depth.o: $(CSRC)/k_depth.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -fmad=false -c $< -o $@
$(OBJDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(OBJDIR)/$*.ptxas.txt || (cat $(OBJDIR)/$*.ptxas.txt; exit 1)

$(PKG)/libisocull_b200.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJS) -lpthread

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(PKG)/libisocull_b200.so
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
