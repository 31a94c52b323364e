# Builds the C-ABI library paper_2309_14509_b200/libulysses_b200.so for sm_100a.
# (oracle/_ref is not built: the reference is pure Python.)
NVCC    ?= nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr \
           -Xptxas -warn-spills -Iinclude
SRCDIR  := paper_2309_14509_b200/csrc
SRCS    := $(wildcard $(SRCDIR)/*.cu)
OBJS    := $(patsubst $(SRCDIR)/%.cu,build/%.o,$(SRCS))
HDRS    := $(wildcard $(SRCDIR)/*.cuh) include/ulysses_b200.h
LIB     := paper_2309_14509_b200/libulysses_b200.so

all: $(LIB)

build/%.o: $(SRCDIR)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart_static -ldl -lrt -lpthread

sass: $(LIB)
	cuobjdump -sass $(LIB) > build/sass.txt

clean:
	rm -rf build $(LIB)

.PHONY: all clean sass

# profiling build with pipeline timestamps (tools/trace_bwd.py); never shipped
TRACE_LIB := build/trace/libulysses_b200_trace.so
trace: $(SRCS) $(HDRS)
	@mkdir -p build/trace
	$(NVCC) $(NVFLAGS) -DUL_TRACE -shared -o $(TRACE_LIB) $(SRCS) -lcudart_static -ldl -lrt -lpthread
.PHONY: trace
