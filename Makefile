# Builds the B200 library in-tree (travels to the GPU box with the snapshot).
#   make            -> paper_2504_12471_b200/libd2ft_b200.so + oracle/_build/liboracle.so
#   make ref        -> also oracle/_ref/libd2ft_ref.so (needs /root/reference)
#   make OBJDIR=build/var/x/obj LIB=build/var/x/libd2ft_b200.so EXTRA=-D...  -> experiment build
#                      (load it with D2FT_B200_LIB=...)
NVCC     ?= /usr/local/cuda/bin/nvcc
PKG      := paper_2504_12471_b200
CSRC     := $(PKG)/csrc
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall \
            --expt-relaxed-constexpr -Iinclude -Xptxas -v $(EXTRA)
OBJDIR   ?= build/obj
SRCS     := $(wildcard $(CSRC)/*.cu)
OBJS     := $(patsubst $(CSRC)/%.cu,$(OBJDIR)/%.o,$(SRCS))
HDRS     := $(wildcard $(CSRC)/*.cuh) include/d2ft_b200.h
LIB      ?= $(PKG)/libd2ft_b200.so
# GEMM self-test hooks (include/d2ft_b200_testing.h): a separate library for
# tests/test_gemm_gpu.py, linked against the product library
TESTLIB  := $(PKG)/libd2ft_b200_testing.so

.PHONY: all ref oracle clean
all: $(LIB) $(TESTLIB) oracle

$(OBJDIR)/testing/%.o: $(CSRC)/testing/%.cu $(HDRS) include/d2ft_b200_testing.h
	@mkdir -p $(OBJDIR)/testing
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJDIR)/testing/$*.ptxas.log || (cat $(OBJDIR)/testing/$*.ptxas.log; exit 1)

$(TESTLIB): $(OBJDIR)/testing/gemm_testing.o $(LIB)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJDIR)/testing/gemm_testing.o -L$(PKG) -ld2ft_b200 -lcuda \
	    -Xlinker -rpath -Xlinker '$$ORIGIN'

$(OBJDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJDIR)/$*.ptxas.log || (cat $(OBJDIR)/$*.ptxas.log; exit 1)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcuda -ldl

oracle:
	$(MAKE) -s -C oracle

ref: all
	$(MAKE) -s -j8 -C oracle ref

clean:
	rm -rf build $(LIB) $(TESTLIB)
	$(MAKE) -s -C oracle clean
