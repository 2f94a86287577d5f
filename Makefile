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
CXX_SRCS  := $(wildcard $(SRC)/host/*.cpp)
CXX_OBJS  := $(patsubst $(SRC)/%.cpp,$(OBJDIR)/%.o,$(CXX_SRCS))
CUDA_HOME ?= /usr/local/cuda
HDRS      := $(wildcard $(SRC)/*.cuh) $(wildcard $(SRC)/*.h) include/gnsb.h $(wildcard include/gnstk/*.hpp)

all: lib oracle cpptest

lib: $(LIBDIR)/libgnsb.so

$(OBJDIR)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; false)

# host-only C++ (the gnstk drop-in shim over the C ABI)
$(OBJDIR)/%.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(dir $@)
	g++ -O2 -std=c++20 -fPIC -Iinclude -I$(CUDA_HOME)/include -c $< -o $@

$(LIBDIR)/libgnsb.so: $(CU_OBJS) $(CXX_OBJS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared -o $@ $(CU_OBJS) $(CXX_OBJS) -lrt -ldl -lpthread

oracle:
	$(MAKE) -C oracle

# C++ drop-in test (links the product library; runs on a GPU box)
cpptest: tests/cpp/test_dropin

tests/cpp/test_dropin: tests/cpp/test_dropin.cpp $(LIBDIR)/libgnsb.so $(wildcard include/gnstk/*.hpp)
	g++ -O2 -std=c++20 -Iinclude -o $@ $< -L$(LIBDIR) -lgnsb -Wl,-rpath,'$$ORIGIN/../../$(LIBDIR)'

clean:
	rm -rf build $(LIBDIR)/libgnsb.so
	$(MAKE) -C oracle clean

.PHONY: all lib oracle cpptest clean
