#include "graph.hpp"

#include <algorithm>
#include <map>
#include <set>

#include "common.hpp"
#include "fusion.hpp"
#include "textdoc.hpp"

namespace xlf {

const char* to_string(LayerKind k) {
    switch (k) {
    case LayerKind::conv: return "conv";
    case LayerKind::pool: return "pool";
    case LayerKind::relu: return "relu";
    case LayerKind::add: return "add";
    case LayerKind::concat: return "concat";
    }
    return "?";
}

const Layer* Graph::find_layer(const std::string& n) const {
    for (const Layer& l : layers)
        if (l.name == n) return &l;
    return nullptr;
}
Layer* Graph::find_layer(const std::string& n) {
    for (Layer& l : layers)
        if (l.name == n) return &l;
    return nullptr;
}
const GraphInput* Graph::find_input(const std::string& n) const {
    for (const GraphInput& i : inputs)
        if (i.name == n) return &i;
    return nullptr;
}
bool Graph::shapes_inferred() const {
    return std::all_of(layers.begin(), layers.end(), [](const Layer& l) { return l.out_shape.has_value(); });
}
TensorShape Graph::shape_of(const std::string& n) const {
    if (const GraphInput* i = find_input(n)) return i->shape;
    const Layer* l = find_layer(n);
    if (!l || !l->out_shape) fail(ErrorKind::internal, "no inferred shape for '" + n + "'");
    return *l->out_shape;
}
std::vector<std::string> Graph::consumers_of(const std::string& n) const {
    std::vector<std::string> r;
    for (const Layer& l : layers)
        if (std::find(l.inputs.begin(), l.inputs.end(), n) != l.inputs.end()) r.push_back(l.name);
    return r;
}
bool Graph::is_output(const std::string& n) const {
    return std::find(outputs.begin(), outputs.end(), n) != outputs.end();
}

int conv_out_dim(int in, int kernel, int pad, int stride) { return (in + 2 * pad - kernel) / stride + 1; }

namespace {

TensorShape read_shape(const td::Node& n) {
    auto v = n.ints();
    if (v.size() != 3) fail(ErrorKind::parse, "shape must be [channels, height, width]", n.line);
    TensorShape s{int(v[0]), int(v[1]), int(v[2])};
    if (s.channels < 1 || s.height < 1 || s.width < 1) fail(ErrorKind::parse, "shape dimensions must be >= 1", n.line);
    return s;
}

ConvParams read_conv(const td::Node& sec) {
    ConvParams c;
    c.out_channels = int(sec.need("out_channels").integer());
    auto k = sec.need("kernel").ints();
    if (k.size() == 1) c.kernel_h = c.kernel_w = int(k[0]);
    else if (k.size() == 2) c.kernel_h = int(k[0]), c.kernel_w = int(k[1]);
    else fail(ErrorKind::parse, "conv kernel must be [kh, kw]", sec.line);
    c.pad = int(sec.int_or("pad", 0));
    c.stride = int(sec.int_or("stride", 1));
    c.group = int(sec.int_or("group", 1));
    c.has_bias = sec.bool_or("bias", true);
    const std::string act = sec.str_or("activation", "none");
    if (act == "relu") c.activation = Activation::relu;
    else if (act != "none") fail(ErrorKind::parse, "unknown activation '" + act + "'", sec.line);
    if (c.out_channels < 1) fail(ErrorKind::parse, "out_channels must be >= 1", sec.line);
    if (c.kernel_h < 1 || c.kernel_w < 1) fail(ErrorKind::parse, "kernel dimensions must be >= 1", sec.line);
    if (c.stride < 1) fail(ErrorKind::parse, "stride must be >= 1", sec.line);
    if (c.pad < 0) fail(ErrorKind::parse, "pad must be >= 0", sec.line);
    if (c.group < 1) fail(ErrorKind::parse, "group must be >= 1", sec.line);
    return c;
}

PoolParams read_pool(const td::Node& sec) {
    PoolParams p;
    const std::string kind = sec.need("pool").str();
    if (kind == "max") p.kind = PoolKind::max;
    else if (kind == "avg") p.kind = PoolKind::avg;
    else fail(ErrorKind::parse, "pool kind must be max or avg", sec.line);
    p.kernel = int(sec.need("kernel").integer());
    p.stride = int(sec.int_or("stride", 1));
    p.pad = int(sec.int_or("pad", 0));
    if (p.kernel < 1 || p.stride < 1 || p.pad < 0) fail(ErrorKind::parse, "bad pool parameters", sec.line);
    return p;
}

LayerKind read_kind(const td::Node& n) {
    const std::string v = n.str();
    if (v == "conv") return LayerKind::conv;
    if (v == "pool") return LayerKind::pool;
    if (v == "relu") return LayerKind::relu;
    if (v == "add") return LayerKind::add;
    if (v == "concat") return LayerKind::concat;
    fail(ErrorKind::parse, "unknown layer kind '" + v + "'", n.line);
}

// Names resolve, arities hold, no cycles (graph.cpp:152-217 semantics).
void check_structure(const Graph& g) {
    std::set<std::string> names;
    auto bad = [&](const Layer* l, const std::string& m) {
        fail(ErrorKind::parse, (l ? l->name + ": " : std::string()) + m, l ? l->line : 0);
    };
    for (const GraphInput& i : g.inputs)
        if (!names.insert(i.name).second) fail(ErrorKind::parse, i.name + ": duplicate name");
    for (const Layer& l : g.layers)
        if (!names.insert(l.name).second) bad(&l, "duplicate layer name");
    for (const Layer& l : g.layers) {
        for (const std::string& in : l.inputs)
            if (!g.find_input(in) && !g.find_layer(in)) bad(&l, "references missing producer '" + in + "'");
        const size_t n = l.inputs.size();
        if ((l.kind == LayerKind::conv || l.kind == LayerKind::pool || l.kind == LayerKind::relu) && n != 1)
            bad(&l, std::string(to_string(l.kind)) + " requires exactly 1 input");
        if (l.kind == LayerKind::add && n != 2) bad(&l, "add requires exactly 2 inputs");
        if (l.kind == LayerKind::concat && n < 2) bad(&l, "concat requires >= 2 inputs");
        if (l.conv && l.conv->out_channels % l.conv->group != 0) bad(&l, "out_channels not divisible by group");
    }
    for (const std::string& o : g.outputs)
        if (!g.find_layer(o) && !g.find_input(o)) fail(ErrorKind::parse, o + ": output references missing layer");
    topo_order(g);  // throws on a cycle
}

}  // namespace

Graph parse_graph(const std::string& text) {
    td::Node doc = td::parse(text);
    Graph g;
    g.name = doc.need("name").str();
    for (const td::Node* in : doc.all("input")) g.inputs.push_back({in->need("name").str(), read_shape(in->need("shape"))});
    if (g.inputs.empty()) fail(ErrorKind::parse, "graph declares no inputs");
    for (const td::Node* ln : doc.all("layer")) {
        Layer l;
        l.line = ln->line;
        l.name = ln->need("name").str();
        l.kind = read_kind(ln->need("kind"));
        l.inputs = ln->need("inputs").values;
        if (l.kind == LayerKind::conv) l.conv = read_conv(*ln);
        if (l.kind == LayerKind::pool) l.pool = read_pool(*ln);
        g.layers.push_back(std::move(l));
    }
    for (const td::Node* o : doc.all("output")) g.outputs.push_back(o->str());
    if (g.outputs.empty()) fail(ErrorKind::parse, "graph declares no outputs");
    try {
        check_structure(g);
    } catch (const Error& e) {
        if (e.kind() == ErrorKind::validation) fail(ErrorKind::parse, e.what());
        throw;
    }
    return g;
}

std::string serialize_graph(const Graph& g) {
    td::Node doc;
    doc.children.push_back(td::leaf("name", g.name));
    for (const GraphInput& i : g.inputs) {
        td::Node s = td::branch("input");
        s.children.push_back(td::leaf("name", i.name));
        s.children.push_back(td::leaf_ints("shape", {i.shape.channels, i.shape.height, i.shape.width}));
        doc.children.push_back(std::move(s));
    }
    for (const Layer& l : g.layers) {
        td::Node s = td::branch("layer");
        s.children.push_back(td::leaf("name", l.name));
        s.children.push_back(td::leaf("kind", std::string(to_string(l.kind))));
        s.children.push_back(td::leaf_list("inputs", l.inputs));
        if (l.conv) {
            const ConvParams& c = *l.conv;
            s.children.push_back(td::leaf("out_channels", (long long)c.out_channels));
            s.children.push_back(td::leaf_ints("kernel", {c.kernel_h, c.kernel_w}));
            s.children.push_back(td::leaf("pad", (long long)c.pad));
            s.children.push_back(td::leaf("stride", (long long)c.stride));
            s.children.push_back(td::leaf("group", (long long)c.group));
            s.children.push_back(td::leaf("bias", std::string(c.has_bias ? "true" : "false")));
            s.children.push_back(td::leaf("activation", std::string(c.activation == Activation::relu ? "relu" : "none")));
        }
        if (l.pool) {
            const PoolParams& p = *l.pool;
            s.children.push_back(td::leaf("pool", std::string(p.kind == PoolKind::max ? "max" : "avg")));
            s.children.push_back(td::leaf("kernel", (long long)p.kernel));
            s.children.push_back(td::leaf("stride", (long long)p.stride));
            s.children.push_back(td::leaf("pad", (long long)p.pad));
        }
        doc.children.push_back(std::move(s));
    }
    for (const std::string& o : g.outputs) doc.children.push_back(td::leaf("output", o));
    return td::serialize(doc);
}

std::vector<const Layer*> topo_order(const Graph& g) {
    std::map<std::string, int> pending;
    for (const Layer& l : g.layers) {
        int d = 0;
        for (const std::string& in : l.inputs) d += g.find_layer(in) != nullptr;
        pending[l.name] = d;
    }
    std::vector<const Layer*> order;
    std::vector<char> done(g.layers.size(), 0);
    while (order.size() < g.layers.size()) {
        size_t pick = g.layers.size();
        for (size_t i = 0; i < g.layers.size(); ++i)
            if (!done[i] && pending[g.layers[i].name] == 0) { pick = i; break; }
        if (pick == g.layers.size()) fail(ErrorKind::validation, "graph contains a cycle");
        done[pick] = 1;
        const Layer& l = g.layers[pick];
        order.push_back(&l);
        for (const Layer& c : g.layers)
            if (std::find(c.inputs.begin(), c.inputs.end(), l.name) != c.inputs.end()) --pending[c.name];
    }
    return order;
}

Graph infer_shapes(const Graph& g0) {
    Graph g = g0;
    for (const Layer* lp : topo_order(g0)) {
        Layer& l = *g.find_layer(lp->name);
        auto in = [&](size_t i) { return g.shape_of(l.inputs[i]); };
        auto why = [&](const std::string& m) { fail(ErrorKind::validation, l.name + ": " + m, l.line); };
        TensorShape s;
        switch (l.kind) {
        case LayerKind::conv: {
            ConvParams& c = *l.conv;
            const TensorShape x = in(0);
            c.in_channels = x.channels;
            if (c.in_channels % c.group) why("input channels " + std::to_string(c.in_channels) + " not divisible by group " + std::to_string(c.group));
            if (c.out_channels % c.group) why("out_channels not divisible by group");
            s = {c.out_channels, conv_out_dim(x.height, c.kernel_h, c.pad, c.stride), conv_out_dim(x.width, c.kernel_w, c.pad, c.stride)};
            if (s.height < 1 || s.width < 1) why("non-positive output dimension");
            break;
        }
        case LayerKind::pool: {
            const PoolParams& p = *l.pool;
            const TensorShape x = in(0);
            s = {x.channels, conv_out_dim(x.height, p.kernel, p.pad, p.stride), conv_out_dim(x.width, p.kernel, p.pad, p.stride)};
            if (s.height < 1 || s.width < 1) why("non-positive output dimension");
            break;
        }
        case LayerKind::relu: s = in(0); break;
        case LayerKind::add:
            if (!(in(0) == in(1))) why("add inputs have different shapes");
            s = in(0);
            break;
        case LayerKind::concat: {
            s = in(0);
            s.channels = 0;
            for (size_t i = 0; i < l.inputs.size(); ++i) {
                const TensorShape x = in(i);
                if (x.height != s.height || x.width != s.width) why("concat inputs differ in height/width");
                s.channels += x.channels;
            }
            break;
        }
        }
        l.out_shape = s;
    }
    return g;
}

Graph prepare_graph(const std::string& text) { return fold_elementwise(infer_shapes(parse_graph(text))); }

}  // namespace xlf
