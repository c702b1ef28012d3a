# libmcf.so (sm_100a) + the CPU oracle.  `python -c "import __graft_entry__ as g; g.build()"`
# runs the same recipe.
NVCC ?= nvcc
MAKEFLAGS += -j8
PKG := paper_1108_2580_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
NVFLAGS := -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
           -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr

all: $(PKG)/libmcf.so oracle

OBJ := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRC))
HDR := $(wildcard $(PKG)/csrc/*.cuh) include/mcf.h

# one object per translation unit (compiled in parallel); ptxas -v output
# (registers / spills per kernel) goes to build/<unit>.ptxas.log
build/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(PKG)/libmcf.so: $(OBJ)
	$(NVCC) -gencode arch=compute_100a,code=sm_100a -shared -o $@ $(OBJ) -ldl

# micro-benchmarks used for the roofline peaks (profiles/fp32_peak.json)
MICRO := $(patsubst %.cu,%,$(wildcard tools/micro/*.cu))
micro: $(MICRO)
tools/micro/%: tools/micro/%.cu
	$(NVCC) -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o $@ $<

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -f $(PKG)/libmcf.so oracle/liboracle.so build/*.o

.PHONY: all oracle clean micro
