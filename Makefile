# Build the C-ABI shared library for sm_100a (B200).  `python -c "import __graft_entry__ as g; g.build()"`
# runs the same recipe.
NVCC    ?= nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude
SRC     := paper_2401_10089_b200/csrc
OUT     := paper_2401_10089_b200/_build
OBJS    := $(OUT)/lgm_api.o $(OUT)/lgm_grid.o $(OUT)/lgm_spectrum.o
LIB     := $(OUT)/liblogmpoly_b200.so

all: $(LIB)

$(OUT)/%.o: $(SRC)/%.cu $(wildcard $(SRC)/*.cuh $(SRC)/*.h) include/logmpoly_b200.h
	@mkdir -p $(OUT)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

clean:
	rm -rf $(OUT)

.PHONY: all clean

# phase-profiling variant (clock64 per Algorithm-1 phase; tools/phase_prof.py)
PROF := $(OUT)/liblogmpoly_b200_prof.so
prof: $(PROF)
$(PROF): $(SRC)/lgm_api.cu $(SRC)/lgm_grid.cu $(wildcard $(SRC)/*.cuh $(SRC)/*.h) include/logmpoly_b200.h
	@mkdir -p $(OUT)
	$(NVCC) $(NVFLAGS) -DLGM_PHASE_PROF -c $(SRC)/lgm_api.cu -o $(OUT)/lgm_api_prof.o
	$(NVCC) $(NVFLAGS) -DLGM_PHASE_PROF -c $(SRC)/lgm_grid.cu -o $(OUT)/lgm_grid_prof.o
	$(NVCC) $(ARCH) -shared -o $@ $(OUT)/lgm_api_prof.o $(OUT)/lgm_grid_prof.o $(OUT)/lgm_spectrum.o
.PHONY: prof

# A/B variants: make variant V=mb10 VFLAGS=-DLGM_F32_MINB=10  (tools/time_lib.py with LGM_LIB)
variant:
	@mkdir -p $(OUT)/var
	$(NVCC) $(NVFLAGS) $(VFLAGS) -c $(SRC)/lgm_api.cu -o $(OUT)/var/lgm_api_$(V).o
	$(NVCC) $(ARCH) -shared -o $(OUT)/var/liblogmpoly_b200_$(V).so $(OUT)/var/lgm_api_$(V).o $(OUT)/lgm_grid.o $(OUT)/lgm_spectrum.o
.PHONY: variant

# A/B variants of the grid engine: make gvariant V=rt64 VFLAGS=-DG2_RT=64
gvariant:
	@mkdir -p $(OUT)/var
	$(NVCC) $(NVFLAGS) $(VFLAGS) -c $(SRC)/lgm_grid.cu -o $(OUT)/var/lgm_grid_$(V).o
	$(NVCC) $(ARCH) -shared -o $(OUT)/var/liblogmpoly_b200_$(V).so $(OUT)/lgm_api.o $(OUT)/var/lgm_grid_$(V).o $(OUT)/lgm_spectrum.o
.PHONY: gvariant
