// oracle/ref_tool.cpp -- TEST INFRASTRUCTURE ONLY.  Command-line access to the
// unmodified reference for outputs that go through C++ iostreams (the field
// dump, weather.cpp:251-269), which must run in a plain C++ process.
//   ref_tool dump <nx> <ny> <nz> <steps> <field: energy|energy_u|energy_surf|energy_pbl>
#include <cstdlib>
#include <cstring>
#include <iostream>

#include "hft/weather.hpp"

int main(int argc, char** argv) {
    if (argc != 7 || std::strcmp(argv[1], "dump") != 0) {
        std::cerr << "usage: ref_tool dump nx ny nz steps field\n";
        return 2;
    }
    hft::GridConfig c;
    c.nx = std::atoll(argv[2]);
    c.ny = std::atoll(argv[3]);
    c.nz = std::atoll(argv[4]);
    hft::SimState s = hft::run_reference(c, std::atoll(argv[5]));
    std::string f = argv[6];
    const hft::ArrayObject& a = f == "energy" ? s.energy
                                : f == "energy_u" ? s.energy_u
                                : f == "energy_surf" ? s.energy_surf
                                                     : s.energy_pbl;
    hft::dump_field(std::cout, a);
    return 0;
}
