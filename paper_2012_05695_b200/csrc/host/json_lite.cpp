#include "json_lite.hpp"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

namespace ddm::json {

namespace {

struct Parser {
    const std::string& s;
    size_t p = 0;

    [[noreturn]] void fail(const char* what) const {
        throw std::runtime_error(std::string("json: ") + what + " at offset " + std::to_string(p));
    }
    void ws() {
        while (p < s.size() && (s[p] == ' ' || s[p] == '\n' || s[p] == '\r' || s[p] == '\t')) ++p;
    }
    bool lit(const char* w) {
        size_t n = 0;
        while (w[n]) ++n;
        if (s.compare(p, n, w) == 0) {
            p += n;
            return true;
        }
        return false;
    }
    std::string str() {
        if (s[p] != '"') fail("expected string");
        ++p;
        std::string out;
        while (p < s.size() && s[p] != '"') {
            char c = s[p++];
            if (c == '\\') {
                if (p >= s.size()) fail("bad escape");
                const char e = s[p++];
                switch (e) {
                case 'n': out += '\n'; break;
                case 't': out += '\t'; break;
                case 'r': out += '\r'; break;
                case 'b': out += '\b'; break;
                case 'f': out += '\f'; break;
                case 'u': {
                    if (p + 4 > s.size()) fail("bad unicode escape");
                    const unsigned cp = (unsigned)std::strtoul(s.substr(p, 4).c_str(), nullptr, 16);
                    p += 4;
                    if (cp < 0x80) out += char(cp);
                    else if (cp < 0x800) {
                        out += char(0xC0 | (cp >> 6));
                        out += char(0x80 | (cp & 0x3F));
                    } else {
                        out += char(0xE0 | (cp >> 12));
                        out += char(0x80 | ((cp >> 6) & 0x3F));
                        out += char(0x80 | (cp & 0x3F));
                    }
                    break;
                }
                default: out += e;
                }
            } else {
                out += c;
            }
        }
        if (p >= s.size()) fail("unterminated string");
        ++p;
        return out;
    }
    Value val() {
        ws();
        if (p >= s.size()) fail("unexpected end");
        const char c = s[p];
        if (c == '{') {
            ++p;
            Value v = Value::object();
            ws();
            if (s[p] == '}') { ++p; return v; }
            for (;;) {
                ws();
                std::string k = str();
                ws();
                if (s[p] != ':') fail("expected ':'");
                ++p;
                v.obj[k] = val();
                ws();
                if (s[p] == ',') { ++p; continue; }
                if (s[p] == '}') { ++p; return v; }
                fail("expected ',' or '}'");
            }
        }
        if (c == '[') {
            ++p;
            Value v = Value::array();
            ws();
            if (s[p] == ']') { ++p; return v; }
            for (;;) {
                v.arr.push_back(val());
                ws();
                if (s[p] == ',') { ++p; continue; }
                if (s[p] == ']') { ++p; return v; }
                fail("expected ',' or ']'");
            }
        }
        if (c == '"') return Value::string(str());
        if (lit("null")) return Value::null();
        if (lit("true")) { Value v; v.kind = Value::Kind::Bool; v.b = true; return v; }
        if (lit("false")) { Value v; v.kind = Value::Kind::Bool; return v; }
        // number
        size_t q = p;
        bool integral = true;
        if (s[q] == '-') ++q;
        while (q < s.size()) {
            const char d = s[q];
            if (d >= '0' && d <= '9') { ++q; continue; }
            if (d == '.' || d == 'e' || d == 'E' || d == '+' || d == '-') { integral = false; ++q; continue; }
            break;
        }
        if (q == p) fail("unexpected character");
        const std::string tok = s.substr(p, q - p);
        p = q;
        if (integral) return Value::integer(std::strtoll(tok.c_str(), nullptr, 10));
        return Value::number(std::strtod(tok.c_str(), nullptr));
    }
};

void emit(const Value& v, std::string& out, int indent, int depth) {
    auto nl = [&](int d) {
        if (indent < 0) return;
        out += '\n';
        out.append((size_t)(indent * d), ' ');
    };
    switch (v.kind) {
    case Value::Kind::Null: out += "null"; break;
    case Value::Kind::Bool: out += v.b ? "true" : "false"; break;
    case Value::Kind::Number: {
        if (v.is_int) {
            out += std::to_string(v.i);
        } else {
            // shortest round-trip form, as nlohmann::json prints (0.1 -> "0.1", not
            // "0.10000000000000001")
            char buf[64];
            for (int prec = 15; prec <= 17; ++prec) {
                std::snprintf(buf, sizeof buf, "%.*g", prec, v.num);
                if (prec == 17 || std::strtod(buf, nullptr) == v.num) break;
            }
            std::string t = buf;
            if (t.find_first_of(".eEn") == std::string::npos) t += ".0";
            out += t;
        }
        break;
    }
    case Value::Kind::String: {
        out += '"';
        for (char c : v.str) {
            if (c == '"' || c == '\\') { out += '\\'; out += c; }
            else if (c == '\n') out += "\\n";
            else out += c;
        }
        out += '"';
        break;
    }
    case Value::Kind::Array: {
        out += '[';
        bool first = true;
        for (const auto& e : v.arr) {
            if (!first) out += ',';
            first = false;
            nl(depth + 1);
            emit(e, out, indent, depth + 1);
        }
        if (!v.arr.empty()) nl(depth);
        out += ']';
        break;
    }
    case Value::Kind::Object: {
        out += '{';
        bool first = true;
        for (const auto& [k, e] : v.obj) {
            if (!first) out += ',';
            first = false;
            nl(depth + 1);
            emit(Value::string(k), out, indent, depth + 1);
            out += indent < 0 ? ":" : ": ";
            emit(e, out, indent, depth + 1);
        }
        if (!v.obj.empty()) nl(depth);
        out += '}';
        break;
    }
    }
}

}  // namespace

const Value& Value::at(const std::string& k) const {
    if (kind != Kind::Object) throw std::runtime_error("json: not an object");
    auto it = obj.find(k);
    if (it == obj.end()) throw std::runtime_error("json: missing key '" + k + "'");
    return it->second;
}

std::int64_t Value::as_int() const {
    if (kind != Kind::Number) throw std::runtime_error("json: not a number");
    if (is_int) return i;
    if (std::floor(num) != num) throw std::runtime_error("json: not an integer");
    return (std::int64_t)num;
}

double Value::as_double() const {
    if (kind != Kind::Number) throw std::runtime_error("json: not a number");
    return is_int ? double(i) : num;
}

const std::string& Value::as_string() const {
    if (kind != Kind::String) throw std::runtime_error("json: not a string");
    return str;
}

std::vector<std::int64_t> Value::as_int_vector() const {
    if (kind != Kind::Array) throw std::runtime_error("json: not an array");
    std::vector<std::int64_t> out;
    out.reserve(arr.size());
    for (const auto& e : arr) out.push_back(e.as_int());
    return out;
}

Value parse(const std::string& text) {
    Parser ps{text};
    Value v = ps.val();
    ps.ws();
    if (ps.p != text.size()) ps.fail("trailing characters");
    return v;
}

std::string dump(const Value& v, int indent) {
    std::string out;
    emit(v, out, indent, 0);
    return out;
}

}  // namespace ddm::json
