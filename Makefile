# Build of libfxg.so (sm_100a CUDA kernels + C ABI + C++ engine layer) and the
# test-only oracles.  `python -c "import __graft_entry__ as g; g.build()"` runs this.
NVCC     ?= nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
PKG      := paper_2603_12016_b200
SRC      := $(PKG)/csrc
OBJ      := $(PKG)/build
LIBDIR   := $(PKG)/lib
LIB      := $(LIBDIR)/libfxg.so
NVFLAGS  := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Iinclude -I$(SRC) \
            --expt-relaxed-constexpr -Xptxas -warn-spills $(FXG_DEFS)
CXXFLAGS := -O3 -std=c++20 -fPIC -Wall -Wextra -Iinclude -I$(SRC) -I/usr/local/cuda/include

CU_SRCS  := $(SRC)/fx_scan.cu $(SRC)/fx_roi_s.cu $(SRC)/fx_roi_b.cu $(SRC)/fx_roi_t.cu $(SRC)/fx_capi.cu $(SRC)/fx_multi.cu $(SRC)/fx_wide.cu
CXX_SRCS := $(SRC)/fx_host.cpp $(SRC)/engine.cpp $(SRC)/fx_pack.cpp
CU_OBJS  := $(patsubst $(SRC)/%.cu,$(OBJ)/%.o,$(CU_SRCS))
CXX_OBJS := $(patsubst $(SRC)/%.cpp,$(OBJ)/%.o,$(CXX_SRCS))
HDRS     := $(wildcard $(SRC)/*.cuh) $(wildcard $(SRC)/*.hpp) $(wildcard include/*.h) \
            $(wildcard include/featurex_gpu/*.hpp)

.PHONY: all lib oracle ref synth clean
all: lib oracle synth

# bench / test tooling (synthetic inputs), not linked into libfxg.so
SYNTH := tools/synth/_build/libfxsynth.so
synth: $(SYNTH)
$(SYNTH): tools/synth/fx_synth.cpp
	@mkdir -p $(dir $@)
	g++ -O2 -std=c++20 -fPIC -shared -Wall -Wextra -o $@ $<

lib: $(LIB)

$(OBJ)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJ)/%.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJ)
	g++ $(CXXFLAGS) -c $< -o $@

$(LIB): $(CU_OBJS) $(CXX_OBJS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $^ -lpthread -ldl -lrt

oracle:
	$(MAKE) -C oracle oracle

ref:
	$(MAKE) -C oracle ref

clean:
	rm -rf $(OBJ) $(LIBDIR) tools/synth/_build
