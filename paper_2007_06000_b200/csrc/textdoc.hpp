// Reader/writer for the reference's structured-text documents (graphs,
// devices, plans): `key value...` lines and `key { ... }` sections, `#`
// comments, brackets and commas as decoration.  Format as specified by the
// reference (include/xlfuse/textdoc.hpp:14-60); implementation is our own.
#pragma once

#include <string>
#include <vector>

namespace xlf::td {

struct Node {
    std::string key;
    std::vector<std::string> values;
    std::vector<Node> children;
    bool section = false;
    int line = 0;

    const Node* find(const std::string& k) const;
    std::vector<const Node*> all(const std::string& k) const;
    const Node& need(const std::string& k) const;

    std::string str() const;
    long long integer() const;
    double real() const;
    bool boolean() const;
    std::vector<long long> ints() const;

    std::string str_or(const std::string& k, const std::string& d) const;
    long long int_or(const std::string& k, long long d) const;
    bool bool_or(const std::string& k, bool d) const;
};

// A document is a nameless root section.
Node parse(const std::string& text);
std::string serialize(const Node& root);

Node leaf(const std::string& key, const std::string& v);
Node leaf(const std::string& key, long long v);
Node leaf(const std::string& key, double v);
Node leaf_list(const std::string& key, const std::vector<std::string>& v);
Node leaf_ints(const std::string& key, const std::vector<long long>& v);
Node branch(const std::string& key);

}  // namespace xlf::td
