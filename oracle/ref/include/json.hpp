// TEST INFRASTRUCTURE ONLY — NOT nlohmann/json.
//
// The reference vendors nlohmann/json as proj/vendor/json.hpp, which is
// git-ignored and absent. bench.hpp and report_json.hpp include it;
// they are outside the hot path but the reference's umbrella header (mvsk.hpp,
// included by its test helpers) pulls them in. This stand-in provides the
// document model those headers and test_solver.cpp use (objects, arrays,
// numbers, strings, bools; operator[], contains, at, get<T>, value, size,
// iteration, comparisons with strings) so they compile unmodified. Text parsing
// is not provided: operator>> throws json::exception.
#pragma once

#include <cstdint>
#include <initializer_list>
#include <istream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace nlohmann {

class json {
public:
    enum class kind { null, boolean, number, string, array, object };
    struct exception : std::runtime_error {
        using std::runtime_error::runtime_error;
    };

    json() = default;
    json(std::nullptr_t) {}
    json(bool b) : k_(kind::boolean), b_(b) {}
    template <class T, typename std::enable_if<std::is_arithmetic<T>::value && !std::is_same<T, bool>::value, int>::type = 0>
    json(T x) : k_(kind::number), num_(static_cast<double>(x)) {}
    json(const std::string& s) : k_(kind::string), s_(s) {}
    json(const char* s) : k_(kind::string), s_(s) {}
    template <class T>
    json(const std::vector<T>& v) : k_(kind::array) {
        for (const auto& x : v) arr_.emplace_back(x);
    }
    json(std::initializer_list<json> il) {
        bool as_object = il.size() > 0;
        for (const auto& e : il)
            if (!(e.k_ == kind::array && e.arr_.size() == 2 && e.arr_[0].k_ == kind::string)) as_object = false;
        if (as_object) {
            k_ = kind::object;
            for (const auto& e : il) obj_.emplace_back(e.arr_[0].s_, e.arr_[1]);
        } else {
            k_ = kind::array;
            arr_.assign(il.begin(), il.end());
        }
    }

    json& operator[](const std::string& key) {
        if (k_ == kind::null) k_ = kind::object;
        if (k_ != kind::object) throw exception("json: operator[] on a non-object");
        for (auto& kv : obj_)
            if (kv.first == key) return kv.second;
        obj_.emplace_back(key, json());
        return obj_.back().second;
    }
    json& operator[](const char* key) { return (*this)[std::string(key)]; }
    const json& operator[](const std::string& key) const { return at(key); }
    const json& operator[](const char* key) const { return at(std::string(key)); }
    const json& at(const std::string& key) const {
        if (k_ == kind::object)
            for (const auto& kv : obj_)
                if (kv.first == key) return kv.second;
        throw exception("json: key not found: " + key);
    }
    bool contains(const std::string& key) const {
        if (k_ != kind::object) return false;
        for (const auto& kv : obj_)
            if (kv.first == key) return true;
        return false;
    }
    template <class T>
    T value(const std::string& key, const T& dflt) const {
        return contains(key) ? at(key).get<T>() : dflt;
    }
    std::string value(const std::string& key, const char* dflt) const {
        return contains(key) ? at(key).get<std::string>() : std::string(dflt);
    }
    template <class T>
    T get() const {
        if constexpr (std::is_same<T, std::string>::value) {
            if (k_ != kind::string) throw exception("json: not a string");
            return s_;
        } else if constexpr (std::is_same<T, bool>::value) {
            if (k_ != kind::boolean) throw exception("json: not a boolean");
            return b_;
        } else {
            if (k_ != kind::number) throw exception("json: not a number");
            return static_cast<T>(num_);
        }
    }
    bool is_array() const { return k_ == kind::array; }
    bool is_object() const { return k_ == kind::object; }
    bool is_string() const { return k_ == kind::string; }
    bool is_number() const { return k_ == kind::number; }
    bool is_null() const { return k_ == kind::null; }
    std::size_t size() const {
        if (k_ == kind::array) return arr_.size();
        if (k_ == kind::object) return obj_.size();
        return k_ == kind::null ? 0 : 1;
    }
    bool empty() const { return size() == 0; }
    std::vector<json>::const_iterator begin() const { return arr_.begin(); }
    std::vector<json>::const_iterator end() const { return arr_.end(); }

    friend bool operator==(const json& a, const char* s) { return a.k_ == kind::string && a.s_ == s; }
    friend bool operator==(const json& a, const std::string& s) { return a.k_ == kind::string && a.s_ == s; }
    friend bool operator==(const json& a, double x) { return a.k_ == kind::number && a.num_ == x; }
    friend std::istream& operator>>(std::istream&, json&) {
        throw exception("json stand-in: text parsing is not provided");
    }

private:
    kind k_ = kind::null;
    bool b_ = false;
    double num_ = 0;
    std::string s_;
    std::vector<json> arr_;
    std::vector<std::pair<std::string, json>> obj_;
};

}  // namespace nlohmann
