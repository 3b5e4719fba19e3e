// Minimal JSON value / parser / writer for the file headers this library exchanges with the
// reference (raw_stack header, partial header, index.json). Not a general JSON library:
// numbers are doubles (integers are kept exactly up to 2^53), objects keep sorted keys.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

namespace ddm::json {

struct Value {
    enum class Kind { Null, Bool, Number, String, Array, Object } kind = Kind::Null;
    bool b = false;
    double num = 0.0;
    bool is_int = false;
    std::int64_t i = 0;
    std::string str;
    std::vector<Value> arr;
    std::map<std::string, Value> obj;

    static Value null() { return {}; }
    static Value integer(std::int64_t v) {
        Value x;
        x.kind = Kind::Number;
        x.is_int = true;
        x.i = v;
        x.num = double(v);
        return x;
    }
    static Value number(double v) {
        Value x;
        x.kind = Kind::Number;
        x.num = v;
        return x;
    }
    static Value string(std::string s) {
        Value x;
        x.kind = Kind::String;
        x.str = std::move(s);
        return x;
    }
    static Value array() {
        Value x;
        x.kind = Kind::Array;
        return x;
    }
    static Value object() {
        Value x;
        x.kind = Kind::Object;
        return x;
    }

    bool has(const std::string& k) const { return kind == Kind::Object && obj.count(k); }
    // accessors throw std::runtime_error on a missing key or wrong kind
    const Value& at(const std::string& k) const;
    std::int64_t as_int() const;
    double as_double() const;
    const std::string& as_string() const;
    std::vector<std::int64_t> as_int_vector() const;
    bool is_null() const { return kind == Kind::Null; }
};

Value parse(const std::string& text);     // throws std::runtime_error
std::string dump(const Value& v, int indent = -1);

}  // namespace ddm::json
