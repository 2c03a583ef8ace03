# Builds the sm_100a C-ABI library of the fast-DQN hot path.
NVCC ?= nvcc
ARCH = -gencode arch=compute_100a,code=sm_100a
NVFLAGS = -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr -rdc=false
SRC = $(wildcard paper_2111_01264_b200/csrc/*.cu)
CSRC = $(wildcard paper_2111_01264_b200/csrc/*.cpp)
HDR = $(wildcard paper_2111_01264_b200/csrc/*.cuh) include/paraq_b200.h
OBJ = $(patsubst paper_2111_01264_b200/csrc/%.cu,build/%.o,$(SRC)) \
      $(patsubst paper_2111_01264_b200/csrc/%.cpp,build/%.host.o,$(CSRC))
LIB = paper_2111_01264_b200/_lib/libparaq_b200.so

all: $(LIB) oracle

build/%.o: paper_2111_01264_b200/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; exit 1)

build/%.host.o: paper_2111_01264_b200/csrc/%.cpp $(HDR)
	@mkdir -p build
	g++ -O2 -std=c++17 -fPIC -ffp-contract=off -c $< -o $@

$(LIB): $(OBJ)
	@mkdir -p paper_2111_01264_b200/_lib
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf build $(LIB)

.PHONY: all oracle clean
