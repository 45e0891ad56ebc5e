# Builds the CUDA C-ABI library in-tree for sm_100a (B200).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
FLAGS := -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC,-ffp-contract=off -Iinclude \
         -Xptxas -v --expt-relaxed-constexpr
LIB := paper_1409_7474_b200/_lib/liblse_b200.so
SRC := paper_1409_7474_b200/csrc/lse_api.cu
HDR := $(wildcard paper_1409_7474_b200/csrc/*.cuh) include/lse_b200.h

all: $(LIB) oracle

$(LIB): $(SRC) $(HDR)
	@mkdir -p $(dir $@)
	$(NVCC) $(FLAGS) -shared -o $@ $(SRC) 2> paper_1409_7474_b200/_lib/ptxas.log || (cat paper_1409_7474_b200/_lib/ptxas.log; false)

# profiling build with per-unit service times (LSE_UNIT_TRACE_FILE=...)
TRACE_LIB := paper_1409_7474_b200/_lib/liblse_b200_trace.so
trace: $(TRACE_LIB)
$(TRACE_LIB): $(SRC) $(HDR)
	@mkdir -p $(dir $@)
	$(NVCC) $(FLAGS) -DLSE_UNIT_TRACE -shared -o $@ $(SRC) 2> /dev/null

# guard-certification build: every fp32 decision also evaluated in fp64
# (lse_check_stats; select with LSE_LIB_PATH)
CHECK_LIB := paper_1409_7474_b200/_lib/liblse_b200_check.so
check: $(CHECK_LIB)
$(CHECK_LIB): $(SRC) $(HDR)
	@mkdir -p $(dir $@)
	$(NVCC) $(FLAGS) -DLSE_CHECK_BOUND -shared -o $@ $(SRC) 2> /dev/null

# resident-kernel phase timing (prints per-phase SM cycles per advance call)
RESTRACE_LIB := paper_1409_7474_b200/_lib/liblse_b200_restrace.so
restrace: $(RESTRACE_LIB) $(TMA_LIB)
$(RESTRACE_LIB): $(SRC) $(HDR)
	@mkdir -p $(dir $@)
	$(NVCC) $(FLAGS) -DLSE_RES_TRACE -shared -o $@ $(SRC) 2> /dev/null

# A/B build: TMA (bulk copy + mbarrier) data ring in the fused pass
TMA_LIB := paper_1409_7474_b200/_lib/liblse_b200_tma.so
tma: $(TMA_LIB)
$(TMA_LIB): $(SRC) $(HDR)
	@mkdir -p $(dir $@)
	$(NVCC) $(FLAGS) -DLSE_TMA_RING=1 -shared -o $@ $(SRC) 2> paper_1409_7474_b200/_lib/ptxas_tma.log

oracle:
	$(MAKE) -C oracle

clean:
	rm -f $(LIB) $(TRACE_LIB) $(CHECK_LIB) $(RESTRACE_LIB) $(TMA_LIB)

.PHONY: all clean oracle trace check restrace tma
