# Build of the B200-native aggmg library (sm_100a) and the CPU oracles.
#   make            -> paper_1403_1649_b200/lib/libaggmg_b200.so + oracle/liboracle.so
#   make ref        -> oracle/_ref/libaggmg_ref.so (needs /root/reference; see oracle/Makefile)
NVCC      ?= /usr/local/cuda/bin/nvcc
HOSTCXX   ?= /usr/bin/g++
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo --fmad=false -std=c++17 -ccbin $(HOSTCXX) \
             -Xcompiler -fPIC,-O2,-Wall,-ffp-contract=off -Xptxas -v,-warn-spills
SRC_DIR   := paper_1403_1649_b200/csrc
OBJ_DIR   := build/obj
LIB       := paper_1403_1649_b200/lib/libaggmg_b200.so
CU_SRCS   := $(wildcard $(SRC_DIR)/*.cu)
CPP_SRCS  := $(wildcard $(SRC_DIR)/*.cpp)
OBJS      := $(patsubst $(SRC_DIR)/%.cu,$(OBJ_DIR)/%.o,$(CU_SRCS)) \
             $(patsubst $(SRC_DIR)/%.cpp,$(OBJ_DIR)/%.cpp.o,$(CPP_SRCS))
HDRS      := $(wildcard $(SRC_DIR)/*.cuh) $(wildcard $(SRC_DIR)/*.hpp) include/aggmg_b200.h

DEMO      := build/cpp_dropin_demo
CLI       := build/aggmg

all: $(LIB) oracle $(DEMO) $(CLI)

# the reference command line (aggmg_main.cpp: generate / solve / bench) over the drop-in header
$(CLI): tools/aggmg_cli.cpp include/aggmg/aggmg.hpp include/aggmg_b200.h $(LIB)
	@mkdir -p build
	$(HOSTCXX) -std=c++20 -O2 -Wall -Iinclude $< -Lpaper_1403_1649_b200/lib -laggmg_b200 \
	  -Wl,-rpath,'$$ORIGIN/../paper_1403_1649_b200/lib' -o $@

# reference-style C++ caller built against the drop-in header include/aggmg/aggmg.hpp
$(DEMO): tools/cpp_dropin_demo.cpp include/aggmg/aggmg.hpp include/aggmg_b200.h $(LIB)
	@mkdir -p build
	$(HOSTCXX) -std=c++20 -O2 -Wall -Iinclude $< -Lpaper_1403_1649_b200/lib -laggmg_b200 \
	  -Wl,-rpath,'$$ORIGIN/../paper_1403_1649_b200/lib' -o $@

$(OBJ_DIR)/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(OBJ_DIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; false)

$(OBJ_DIR)/%.cpp.o: $(SRC_DIR)/%.cpp $(HDRS)
	@mkdir -p $(OBJ_DIR)
	$(HOSTCXX) -std=c++17 -O2 -fPIC -Wall -ffp-contract=off -I/usr/local/cuda/include -c $< -o $@

$(LIB): $(OBJS)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -Xcompiler -fPIC

oracle:
	$(MAKE) -C oracle

ref:
	$(MAKE) -C oracle ref

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all oracle ref clean
