// Prints grasp::records::format_json_double(v) (the records writer's double layout) for each
// double read from stdin (hex float text); tests/test_records_jsonl.py compares the lines with
// the real nlohmann 3.11.3 json(v).dump().
#include "grasp/records.hpp"

#include <cstdlib>
#include <iostream>
#include <string>

int main() {
  std::string tok;
  while (std::cin >> tok) std::cout << grasp::records::format_json_double(std::strtod(tok.c_str(), nullptr)) << "\n";
  return 0;
}
