# Builds the in-tree native library (host compiler + sm_100a kernels) and the
# oracle's C restatement.  `python __graft_entry__.py build` runs the same.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
PKG := paper_2605_14277_b200
LIB := $(PKG)/_lib/libseqcfr_b200.so
# -fmad=false + explicit _rn intrinsics: no FMA contraction anywhere (the
# reference rounds every multiply and add separately).
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -fmad=false -Xcompiler -fPIC,-ffp-contract=off -Xptxas -v
CXXFLAGS := -O3 -std=c++17 -fPIC -ffp-contract=off -Wall
SRC_CU := $(wildcard $(PKG)/csrc/*.cu)
SRC_CPP := $(wildcard $(PKG)/csrc/*.cpp)
HDR := $(wildcard $(PKG)/csrc/*.h $(PKG)/csrc/*.cuh) include/seqcfr_b200.h
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRC_CU)) $(patsubst $(PKG)/csrc/%.cpp,build/%.o,$(SRC_CPP))

all: $(LIB) oracle

build/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

build/%.o: $(PKG)/csrc/%.cpp $(HDR)
	@mkdir -p build
	g++ $(CXXFLAGS) -c $< -o $@

$(LIB): $(OBJ)
	@mkdir -p $(PKG)/_lib
	$(NVCC) -shared $(ARCH) -o $@ $(OBJ) -lcudart

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(PKG)/_lib
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
