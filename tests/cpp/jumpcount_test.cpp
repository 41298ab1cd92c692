// Host-only check of the facade's arbitrary-precision JumpCount (the subset of
// boost::multiprecision::cpp_int that jumpcount.hpp / jump.hpp / polyring.hpp
// use) and of parse_jump_count (jumpcount.hpp:16-47), driven by
// tests/test_facade.py: each stdin line is "op a b" (decimal operands), each
// stdout line the result, compared there with Python's integers.
#include <iostream>
#include <sstream>
#include <string>

#include "ranmar_b200.hpp"

using ranmar::JumpCount;

int main() {
    std::string line;
    while (std::getline(std::cin, line)) {
        std::istringstream in(line);
        std::string op, sa, sb;
        in >> op >> sa >> sb;
        try {
            if (op == "parse") {
                std::cout << ranmar::parse_jump_count(sa).str() << "\n";
                continue;
            }
            if (op == "parseabi") {  // huge counts: the limbs after the period reduction
                const ranmar_jump_count j = ranmar::detail::to_abi(ranmar::parse_jump_count(sa));
                std::cout << j.limb[0] << " " << j.limb[1] << " " << j.limb[2] << " " << j.limb[3] << "\n";
                continue;
            }
            const JumpCount a(sa), b(sb.empty() ? std::string("0") : sb);
            if (op == "add") std::cout << (a + b).str();
            else if (op == "sub") std::cout << (a - b).str();
            else if (op == "mul") std::cout << (a * b).str();
            else if (op == "div") std::cout << (a / b).str();
            else if (op == "mod") std::cout << (a % b).str();
            else if (op == "shl") std::cout << (a << static_cast<unsigned long>(b)).str();
            else if (op == "shr") std::cout << (a >> static_cast<unsigned long>(b)).str();
            else if (op == "cmp") std::cout << (a < b) << (a == b) << (a > b) << (a <= b) << (a >= b);
            else if (op == "msb") std::cout << msb(a);
            else if (op == "bit") std::cout << bit_test(a, static_cast<unsigned>(b));
            else if (op == "u64") std::cout << static_cast<std::uint64_t>(a);
            else if (op == "abi") {  // the 256-bit limbs a jump by a uses (a mod the period)
                const ranmar_jump_count j = ranmar::detail::to_abi(a);
                std::cout << j.limb[0] << " " << j.limb[1] << " " << j.limb[2] << " " << j.limb[3];
            } else std::cout << "?";
        } catch (const std::invalid_argument&) {
            std::cout << "invalid_argument";
        } catch (const std::domain_error&) {
            std::cout << "domain_error";
        }
        std::cout << "\n";
    }
    return 0;
}
