# Top-level build: the product library (CUDA sm_100a + C ABI) and the oracle.
#
#   make            -> paper_2411_00999_b200/lib/libgnsb.so, oracle/liboracle.so,
#                      oracle/_ref/libgnstk_ref.so (when /root/reference exists)
#   make lib        -> product library only
#   make -j         -> parallel (one object per dtype)

NVCC      ?= nvcc
PKG       := paper_2411_00999_b200
SRC       := $(PKG)/csrc
OBJDIR    := build/obj
LIBDIR    := $(PKG)/lib
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-O3 \
             -Xptxas -v -Iinclude $(EXTRA_NVFLAGS)

CU_SRCS   := $(wildcard $(SRC)/*.cu)
CU_OBJS   := $(patsubst $(SRC)/%.cu,$(OBJDIR)/%.o,$(CU_SRCS))
HDRS      := $(wildcard $(SRC)/*.cuh) $(wildcard $(SRC)/*.h) include/gnsb.h

all: lib oracle

lib: $(LIBDIR)/libgnsb.so

$(OBJDIR)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; false)

$(LIBDIR)/libgnsb.so: $(CU_OBJS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared -o $@ $(CU_OBJS) -lrt -ldl -lpthread

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIBDIR)/libgnsb.so
	$(MAKE) -C oracle clean

.PHONY: all lib oracle clean
