#include "textdoc.hpp"

#include <cctype>
#include <cstdio>
#include <cstdlib>
#include <sstream>

#include "common.hpp"

namespace xlf::td {

namespace {

std::string trim(const std::string& s) {
    size_t a = 0, b = s.size();
    while (a < b && std::isspace(static_cast<unsigned char>(s[a]))) ++a;
    while (b > a && std::isspace(static_cast<unsigned char>(s[b - 1]))) --b;
    return s.substr(a, b - a);
}

// Values: whitespace-separated tokens; '[' ']' ',' are separators only.
std::vector<std::string> split_values(const std::string& s, int line) {
    std::vector<std::string> out;
    std::string tok;
    auto flush = [&] {
        if (!tok.empty()) out.push_back(tok), tok.clear();
    };
    for (char ch : s) {
        if (ch == '[' || ch == ']' || ch == ',' || std::isspace(static_cast<unsigned char>(ch))) flush();
        else tok += ch;
    }
    flush();
    if (out.empty()) fail(ErrorKind::parse, "expected a value after key", line);
    return out;
}

void write_node(std::ostringstream& os, const Node& n, int depth) {
    const std::string ind(static_cast<size_t>(depth) * 2, ' ');
    os << ind << n.key;
    if (n.section) {
        os << " {\n";
        for (const Node& c : n.children) write_node(os, c, depth + 1);
        os << ind << "}\n";
        return;
    }
    if (n.values.size() == 1) {
        os << ' ' << n.values[0] << '\n';
        return;
    }
    os << " [";
    for (size_t i = 0; i < n.values.size(); ++i) os << (i ? ", " : "") << n.values[i];
    os << "]\n";
}

}  // namespace

const Node* Node::find(const std::string& k) const {
    for (const Node& c : children)
        if (c.key == k) return &c;
    return nullptr;
}

std::vector<const Node*> Node::all(const std::string& k) const {
    std::vector<const Node*> r;
    for (const Node& c : children)
        if (c.key == k) r.push_back(&c);
    return r;
}

const Node& Node::need(const std::string& k) const {
    const Node* n = find(k);
    if (!n) fail(ErrorKind::parse, (key.empty() ? "document" : "section '" + key + "'") + " is missing required key '" + k + "'", line);
    return *n;
}

std::string Node::str() const {
    if (section || values.size() != 1) fail(ErrorKind::parse, "'" + key + "' must have exactly one value", line);
    return values[0];
}

long long Node::integer() const {
    const std::string s = str();
    char* end = nullptr;
    long long v = std::strtoll(s.c_str(), &end, 10);
    if (end == s.c_str() || *end) fail(ErrorKind::parse, "'" + key + "' is not an integer: " + s, line);
    return v;
}

double Node::real() const {
    const std::string s = str();
    char* end = nullptr;
    double v = std::strtod(s.c_str(), &end);
    if (end == s.c_str() || *end) fail(ErrorKind::parse, "'" + key + "' is not a number: " + s, line);
    return v;
}

bool Node::boolean() const {
    const std::string s = str();
    if (s == "true") return true;
    if (s == "false") return false;
    fail(ErrorKind::parse, "'" + key + "' must be true or false", line);
}

std::vector<long long> Node::ints() const {
    std::vector<long long> r;
    for (const std::string& s : values) {
        char* end = nullptr;
        long long v = std::strtoll(s.c_str(), &end, 10);
        if (end == s.c_str() || *end) fail(ErrorKind::parse, "'" + key + "' holds a non-integer: " + s, line);
        r.push_back(v);
    }
    return r;
}

std::string Node::str_or(const std::string& k, const std::string& d) const {
    const Node* n = find(k);
    return n ? n->str() : d;
}
long long Node::int_or(const std::string& k, long long d) const {
    const Node* n = find(k);
    return n ? n->integer() : d;
}
bool Node::bool_or(const std::string& k, bool d) const {
    const Node* n = find(k);
    return n ? n->boolean() : d;
}

Node parse(const std::string& text) {
    Node root;
    root.section = true;
    std::vector<Node*> open{&root};
    std::istringstream in(text);
    std::string raw;
    int lineno = 0;
    while (std::getline(in, raw)) {
        ++lineno;
        const size_t hash = raw.find('#');
        std::string line = trim(hash == std::string::npos ? raw : raw.substr(0, hash));
        if (line.empty()) continue;
        if (line == "}") {
            if (open.size() == 1) fail(ErrorKind::parse, "unmatched '}'", lineno);
            open.pop_back();
            continue;
        }
        size_t sp = 0;
        while (sp < line.size() && !std::isspace(static_cast<unsigned char>(line[sp]))) ++sp;
        Node n;
        n.key = line.substr(0, sp);
        n.line = lineno;
        const std::string rest = trim(line.substr(sp));
        if (n.key.find_first_of("{}") != std::string::npos)
            fail(ErrorKind::parse, "key '" + n.key + "' must be separated from braces by whitespace", lineno);
        if (rest == "{") {
            n.section = true;
            open.back()->children.push_back(std::move(n));
            open.push_back(&open.back()->children.back());
            continue;
        }
        if (!rest.empty() && rest.back() == '{') fail(ErrorKind::parse, "'{' must be the last token on its line", lineno);
        if (rest.empty()) fail(ErrorKind::parse, "key '" + n.key + "' has no value", lineno);
        n.values = split_values(rest, lineno);
        open.back()->children.push_back(std::move(n));
    }
    if (open.size() > 1) fail(ErrorKind::parse, "section '" + open.back()->key + "' is never closed", open.back()->line);
    return root;
}

std::string serialize(const Node& root) {
    std::ostringstream os;
    for (const Node& c : root.children) write_node(os, c, 0);
    return os.str();
}

Node leaf(const std::string& key, const std::string& v) {
    Node n;
    n.key = key;
    n.values = {v};
    return n;
}
Node leaf(const std::string& key, long long v) { return leaf(key, std::to_string(v)); }
Node leaf(const std::string& key, double v) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return leaf(key, std::string(buf));
}
Node leaf_list(const std::string& key, const std::vector<std::string>& v) {
    Node n;
    n.key = key;
    n.values = v;
    return n;
}
Node leaf_ints(const std::string& key, const std::vector<long long>& v) {
    Node n;
    n.key = key;
    for (long long x : v) n.values.push_back(std::to_string(x));
    return n;
}
Node branch(const std::string& key) {
    Node n;
    n.key = key;
    n.section = true;
    return n;
}

}  // namespace xlf::td
