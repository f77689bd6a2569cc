// C++ side of the ROM-archive format tests (tests/test_archive.py), built
// against the mirrored API (include/mswave/rom_archive.hpp) and the product
// library.  Host only, no device calls.
//   archive_tool copy <src> <dst>   read_rom_archive(src) -> write_rom_archive(dst)
//   archive_tool read <dir>         prints "ok <cells> <ifaces> <sum of ladder entries>"
// Errors print "error <message>" and exit 2 (ConfigError).
#include <cstdio>
#include <string>

#include "mswave/rom_archive.hpp"

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: archive_tool copy <src> <dst> | read <dir>\n");
    return 1;
  }
  const std::string mode = argv[1];
  try {
    mswave::RomArchive ar = mswave::read_rom_archive(argv[2]);
    if (mode == "copy" && argc >= 4) {
      mswave::write_rom_archive(argv[3], ar.roms, ar.basis, ar.opt);
      std::printf("ok\n");
      return 0;
    }
    double sum = 0.0;
    for (const auto& r : ar.roms) {
      for (const auto& L : r.ladder)
        for (long i = 0; i < L.size(); ++i) sum += L.data()[i];
      for (const auto& L : r.ladder_hat)
        for (long i = 0; i < L.size(); ++i) sum += L.data()[i];
    }
    std::printf("ok %zu %zu %.17g\n", ar.roms.size(), ar.basis.S.size(), sum);
    return 0;
  } catch (const mswave::ConfigError& e) {
    std::printf("error %s\n", e.what());
    return 2;
  }
}
