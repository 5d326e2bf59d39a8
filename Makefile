# libfsmc.so: the sm_100a engine behind paper_2503_17405_b200/ (C ABI: include/fsmc.h)
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
# --fmad=false: every fp64 multiply and add rounds once, as numpy does (parity);
# the explicit fma() calls (glibc log restatement, dot products) still fuse.
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 --fmad=false -Xcompiler -fPIC -Xptxas -v $(EXTRA)
CSRC := paper_2503_17405_b200/csrc
BUILD ?= build
LIB ?= paper_2503_17405_b200/libfsmc.so
UNITS := fsmc fam_drmh fam_ess fam_nuts fam_slice logreg_tc gp_chol prior_trmm
OBJS := $(addprefix $(BUILD)/,$(addsuffix .o,$(UNITS)))
HDR := $(wildcard $(CSRC)/*.cuh $(CSRC)/*.h) include/fsmc.h

all: $(LIB) oracle

$(BUILD)/%.o: $(CSRC)/%.cu $(HDR)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $(BUILD)/$*.ptxas.log || (cat $(BUILD)/$*.ptxas.log; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJS)

oracle:
	$(MAKE) -C oracle -s

clean:
	rm -rf $(LIB) $(BUILD) oracle/liboracle.so
.PHONY: all oracle clean

# measured pipe ceilings (fp64 FMA, 64-bit multiply) for the compute roofline
tools/peak_probe: tools/peak_probe.cu
	$(NVCC) $(ARCH) -O3 -o $@ $<
