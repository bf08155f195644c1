// kv_check -- TEST INFRASTRUCTURE: the reference's cfg::KeyValue
// (core/config.cpp, compiled in place) on stdin: prints dump() and hash().
// Optional `set` lines after a `---` separator exercise KeyValue::set(double).
#include <cstdio>
#include <iostream>
#include <sstream>
#include <string>

#include "core/config.hpp"

int main() {
    std::stringstream ss;
    ss << std::cin.rdbuf();
    std::string text = ss.str(), sets;
    const size_t sep = text.find("\n---\n");
    if (sep != std::string::npos) sets = text.substr(sep + 5), text = text.substr(0, sep + 1);
    try {
        zsim::cfg::KeyValue kv = zsim::cfg::KeyValue::parse_text(text);
        std::istringstream in(sets);
        std::string key;
        double v;
        while (in >> key >> v) kv.set(key, v);
        std::cout << kv.dump() << "hash=" << kv.hash() << "\n";
    } catch (const std::exception& e) {
        std::cout << "error: " << e.what() << "\n";
    }
    return 0;
}
