// ir.cpp -- IR text loader of the engine (SPEC S:139 grammar plus the
// U / CU custom-matrix extension, reading R15).  One moment per line, gates separated by
// ';'; header lines "qubits: n", "family: tag", "meta.<k>: v"; '#' starts a comment line.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <sstream>

#include "engine.hpp"

namespace svb {

namespace {

std::string trim(const std::string& s) {
    size_t a = 0, b = s.size();
    while (a < b && std::isspace((unsigned char)s[a])) ++a;
    while (b > a && std::isspace((unsigned char)s[b - 1])) --b;
    return s.substr(a, b - a);
}

bool parse_int_list(const std::string& s, std::vector<int>& out) {
    out.clear();
    std::string tok;
    std::stringstream ss(s);
    while (std::getline(ss, tok, ',')) {
        tok = trim(tok);
        if (tok.empty()) return false;
        for (char c : tok)
            if (!std::isdigit((unsigned char)c)) return false;
        if (tok.size() > 6) return false;
        out.push_back(std::atoi(tok.c_str()));
    }
    return !out.empty();
}

}  // namespace

// SURVEY App. A gate table; R3 fixes the SqrtX/SqrtY global phases.
bool named_gate(const std::string& nm, int& nc, int& k, std::vector<cd>& U) {
    const double r = 0.70710678118654752440;  // fl(1/sqrt 2)
    const cd I(0, 1);
    nc = 0;
    k = 1;
    if (nm == "X") U = {0, 1, 1, 0};
    else if (nm == "Y") U = {0, -I, I, 0};
    else if (nm == "Z") U = {1, 0, 0, -1};
    else if (nm == "H") U = {r, r, r, -r};
    else if (nm == "S") U = {1, 0, 0, I};
    else if (nm == "Sdg") U = {1, 0, 0, -I};
    else if (nm == "T") U = {1, 0, 0, cd(r, r)};
    else if (nm == "Tdg") U = {1, 0, 0, cd(r, -r)};
    else if (nm == "SqrtX") U = {cd(.5, .5), cd(.5, -.5), cd(.5, -.5), cd(.5, .5)};
    else if (nm == "SqrtXdg") U = {cd(.5, -.5), cd(.5, .5), cd(.5, .5), cd(.5, -.5)};
    else if (nm == "SqrtY") U = {cd(.5, .5), cd(-.5, -.5), cd(.5, .5), cd(.5, .5)};
    else if (nm == "SqrtYdg") U = {cd(.5, -.5), cd(.5, -.5), cd(-.5, .5), cd(.5, -.5)};
    else if (nm == "CZ") { nc = 1; U = {1, 0, 0, -1}; }
    else if (nm == "CNOT") { nc = 1; U = {0, 1, 1, 0}; }
    else if (nm == "Toffoli") { nc = 2; U = {0, 1, 1, 0}; }
    else if (nm == "SWAP") { k = 2; U = {1, 0, 0, 0, 0, 0, 1, 0, 0, 1, 0, 0, 0, 0, 0, 1}; }
    else return false;
    return true;
}

static sv_status parse_gate(const std::string& src, int n, int line, Gate& g, std::string& err) {
    auto fail = [&](const std::string& what) {
        err = "line " + std::to_string(line) + ": " + what;
        return SV_ERR_PARSE;
    };
    size_t i = 0;
    while (i < src.size() && (std::isalnum((unsigned char)src[i]) || src[i] == '_')) ++i;
    const std::string name = src.substr(0, i);
    if (name.empty()) return fail("expected a gate name in '" + src + "'");
    std::string rest = src.substr(i);
    g = Gate();
    g.line = line;
    if (name == "U" || name == "CU") {
        const size_t colon = rest.find(':');
        if (colon == std::string::npos) return fail(name + " needs ': matrix'");
        std::string qpart = rest.substr(0, colon);
        std::string mpart = rest.substr(colon + 1);
        if (name == "CU") {
            const size_t bar = qpart.find('|');
            if (bar == std::string::npos) return fail("CU needs 'controls|targets'");
            if (!parse_int_list(qpart.substr(0, bar), g.controls)) return fail("bad CU control list");
            qpart = qpart.substr(bar + 1);
        }
        if (!parse_int_list(qpart, g.targets)) return fail("bad " + name + " target list");
        const int k = (int)g.targets.size();
        if (k > 5) return fail(name + " acts on more than 5 targets");
        const size_t d = (size_t)1 << k;
        std::vector<double> nums;
        const char* p = mpart.c_str();
        for (;;) {
            while (*p == ' ' || *p == '\t') ++p;
            char* e = nullptr;
            const double v = std::strtod(p, &e);
            if (e == p) return fail("bad number in " + name + " matrix");
            nums.push_back(v);
            p = e;
            while (*p == ' ' || *p == '\t') ++p;
            if (*p == ',') { ++p; continue; }
            if (*p == 0) break;
            return fail("unexpected text in " + name + " matrix");
        }
        if (nums.size() != 2 * d * d) return fail(name + " matrix has the wrong size");
        g.U.resize(d * d);
        for (size_t j = 0; j < d * d; ++j) g.U[j] = cd(snap_entry(nums[2 * j]), snap_entry(nums[2 * j + 1]));
    } else {
        int nc, k;
        std::vector<cd> U;
        if (!named_gate(name, nc, k, U)) return fail("unknown gate '" + name + "'");
        std::vector<int> qs;
        if (!parse_int_list(rest, qs)) return fail("bad qubit list for " + name);
        if ((int)qs.size() != nc + k) return fail("wrong qubit count for " + name);
        g.controls.assign(qs.begin(), qs.begin() + nc);
        g.targets.assign(qs.begin() + nc, qs.end());
        g.U = U;
    }
    std::vector<int> all = g.controls;
    all.insert(all.end(), g.targets.begin(), g.targets.end());
    for (size_t a = 0; a < all.size(); ++a) {
        if (all[a] < 0 || all[a] >= n) return fail("qubit " + std::to_string(all[a]) + " out of range");
        for (size_t b = 0; b < a; ++b)
            if (all[a] == all[b]) return fail("duplicate qubit " + std::to_string(all[a]));
    }
    return SV_OK;
}

sv_status parse_ir(const char* text, Circuit& out, std::string& err) {
    out = Circuit();
    if (!text) { err = "null IR text"; return SV_ERR_ARG; }
    std::stringstream ss(text);
    std::string raw;
    int line = 0;
    while (std::getline(ss, raw)) {
        ++line;
        const std::string s = trim(raw);
        if (s.empty() || s[0] == '#') continue;
        if (s.rfind("qubits:", 0) == 0) {
            const std::string v = trim(s.substr(7));
            char* e = nullptr;
            const long n = std::strtol(v.c_str(), &e, 10);
            if (v.empty() || *e || n < 1 || n > 62) {
                err = "line " + std::to_string(line) + ": bad qubit count";
                return SV_ERR_PARSE;
            }
            // one header, before any gate: gates are range-checked against the n in force
            // when they are parsed, so a later (smaller) header would leave them out of range
            if (out.n >= 0) {
                err = "line " + std::to_string(line) + ": repeated 'qubits:' header";
                return SV_ERR_PARSE;
            }
            out.n = (int)n;
            continue;
        }
        if (s.rfind("family:", 0) == 0 || s.rfind("meta.", 0) == 0) continue;
        if (out.n < 0) {
            err = "line " + std::to_string(line) + ": gate before the 'qubits:' header";
            return SV_ERR_PARSE;
        }
        std::stringstream ls(s);
        std::string gtxt;
        while (std::getline(ls, gtxt, ';')) {
            gtxt = trim(gtxt);
            if (gtxt.empty()) continue;
            Gate g;
            const sv_status st = parse_gate(gtxt, out.n, line, g, err);
            if (st != SV_OK) return st;
            out.gates.push_back(std::move(g));
        }
    }
    if (out.n < 0) {
        err = "line " + std::to_string(line) + ": missing 'qubits:' header";
        return SV_ERR_PARSE;
    }
    return SV_OK;
}

}  // namespace svb
