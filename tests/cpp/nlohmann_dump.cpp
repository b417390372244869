// Pins the records writer (host/records.cpp) and the oracle's restatement of nlohmann's dump
// (oracle/records_ref.py) to the real nlohmann/json 3.11.x -- the library the reference's
// records.cpp:65-152 writes with -- using the copy of its single header that ships in this
// image (cudnn_frontend/thirdparty/nlohmann/json.hpp; test-only, not linked into the product).
//   nlohmann_dump lines.jsonl   -> prints json::parse(line).dump() for every line
//   nlohmann_dump --doubles     -> prints json(v).dump() for each double read from stdin (%a hex)
#include <nlohmann/json.hpp>

#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <string>

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "--doubles") {
    std::string tok;
    while (std::cin >> tok) {
      const double v = std::strtod(tok.c_str(), nullptr);
      std::cout << nlohmann::json(v).dump() << "\n";
    }
    return 0;
  }
  std::ifstream in(argv[1]);
  std::string line;
  while (std::getline(in, line)) std::cout << nlohmann::json::parse(line).dump() << "\n";
  return 0;
}
