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

# profiling build with the timeline / per-CTA trace probes compiled in (PQ_LIB selects it)
PLIB = paper_2111_01264_b200/_lib/probes/libparaq_b200.so
POBJ = $(patsubst build/%.o,build/probes/%.o,$(OBJ))
probes: $(PLIB)
build/probes/%.o: paper_2111_01264_b200/csrc/%.cu $(HDR)
	@mkdir -p build/probes
	$(NVCC) $(NVFLAGS) -DPQ_PROBES=1 -c $< -o $@ 2> build/probes/$*.ptxas.log || (cat build/probes/$*.ptxas.log; exit 1)
build/probes/%.host.o: paper_2111_01264_b200/csrc/%.cpp $(HDR)
	@mkdir -p build/probes
	g++ -O2 -std=c++17 -fPIC -ffp-contract=off -c $< -o $@
$(PLIB): $(POBJ)
	@mkdir -p paper_2111_01264_b200/_lib/probes
	$(NVCC) $(ARCH) -shared -o $@ $(POBJ) -lcudart

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
	rm -rf build $(LIB) $(PLIB)

.PHONY: all oracle clean probes
