// tests/cpp/emit_corpus.cpp -- runs the CUDA C++ backend (include/hft_b200/
// emit_cuda_cpp.hpp) over the reference's corpus at BUILD time: the reference's
// own front end parses the .h90 sources, the backend writes one .cu file (a
// build artefact, never committed) and a kernel list.  The Makefile compiles it
// with nvcc for sm_100a; tests/test_emit_gpu.py runs it on the library's fields.
// usage: emit_corpus <corpus dir> <out.cu> <out.txt>
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "hft/parser.hpp"
#include "hft/pipeline.hpp"
#include "hft_b200/emit_cuda_cpp.hpp"

int main(int argc, char** argv) {
    if (argc != 4) {
        std::fprintf(stderr, "usage: %s <corpus dir> <out.cu> <out.txt>\n", argv[0]);
        return 2;
    }
    hft::Diagnostics d;
    std::vector<std::vector<hft::LogicalLine>> files;
    for (const char* f : {"simple_weather.h90", "physics.h90", "diffusion.h90"})
        files.push_back(hft::load_and_merge(std::string(argv[1]) + "/" + f, d).logical);
    hft::ast::Program prog = hft::parse_program(files, d);
    if (!d.ok()) {
        std::fputs(d.render().c_str(), stderr);
        return 1;
    }
    hft::b200::emit::Output out = hft::b200::emit::emit_cuda_cpp(prog, d);
    if (!d.ok()) {
        std::fputs(d.render().c_str(), stderr);
        return 1;
    }
    std::ofstream(argv[2]) << out.source;
    std::ofstream lst(argv[3]);
    for (const auto& k : out.kernels) {
        lst << k.name << " " << k.routine << " " << k.region;
        for (const auto& a : k.arrays) lst << " array:" << a;
        for (const auto& a : k.ints) lst << " int:" << a;
        for (const auto& a : k.reals) lst << " real:" << a;
        lst << "\n";
    }
    return 0;
}
