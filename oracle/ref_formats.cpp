// ref_formats.cpp — the reference's own FLO1 / P4 writers as a command (TEST INFRASTRUCTURE).
//
// Built by `make -C oracle ref` against the UNMODIFIED reference headers.  The writers use
// iostreams, so they run in their own process rather than through the ctypes shim:
//   ref_formats flo <w> <h> <u.f32> <v.f32> <out.flo>   (save_flo, flow.hpp:349-366)
//   ref_formats pbm <w> <h> <mask.u8> <out.pbm>         (save_pbm, pgm.hpp:127-138)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "flowroi/flow.hpp"
#include "flowroi/pgm.hpp"

static std::vector<char> slurp(const char* path) {
    std::ifstream in(path, std::ios::binary);
    return std::vector<char>((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const std::string what = argv[1];
    try {
        if (what == "flo" && argc == 7) {
            flowroi::FlowField f(std::atoi(argv[2]), std::atoi(argv[3]));
            const auto u = slurp(argv[4]), v = slurp(argv[5]);
            if (u.size() != 4 * f.size() || v.size() != 4 * f.size()) return 3;
            std::memcpy(f.u.data(), u.data(), u.size());
            std::memcpy(f.v.data(), v.data(), v.size());
            flowroi::save_flo(f, argv[6]);
            return 0;
        }
        if (what == "pbm" && argc == 6) {
            flowroi::RoiMask m(std::atoi(argv[2]), std::atoi(argv[3]));
            const auto b = slurp(argv[4]);
            if (b.size() != m.size()) return 3;
            std::memcpy(m.bits.data(), b.data(), b.size());
            flowroi::save_pbm(m, argv[5]);
            return 0;
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "%s\n", e.what());
        return 1;
    }
    return 2;
}
