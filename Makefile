# libspt_ffn.so: the sm_100a routed-FFN library (C ABI in include/spt_ffn.h)
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
           --expt-relaxed-constexpr -Iinclude
PKG := paper_2312_10365_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
HDR := $(wildcard $(PKG)/csrc/*.cuh) $(wildcard $(PKG)/csrc/*.h) include/spt_ffn.h
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRC))
LIB := $(PKG)/libspt_ffn.so

all: $(LIB) oracle/libspt_oracle.so

build/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart

oracle/libspt_oracle.so: oracle/spt_oracle.c
	gcc -O2 -fopenmp -fPIC -shared -std=c11 -o $@ $< -lm

sass: $(LIB)
	cuobjdump -sass $(LIB) | grep -oE "UTC[A-Z]*MMA[A-Z0-9.]*|UTMALDG[A-Z0-9.]*|UTMASTG|LDTM[A-Z0-9.]*|HMMA" | sort | uniq -c

clean:
	rm -rf build $(LIB) oracle/libspt_oracle.so

.PHONY: all clean sass
