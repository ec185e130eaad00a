// Access-annotation DSL: parsing and per-superblock region inference.
//
// Grammar and semantics are those of the reference (proj/src/annotation.cpp:105-391 for the
// parser, :440-517 for evaluation, :524-538 for the write-overlap rule):
//   annotation := binding (',' binding)* '=>' [access (',' access)*]
//   binding    := ('global'|'block'|'local') (ident | '[' ident (',' ident)* ']')
//   access     := mode ident '[' index (',' index)* ']'
//   mode       := 'read' | 'write' | 'readwrite' | 'reduce' '(' ('+'|'*'|'min'|'max') ')'
//   index      := expr | [expr] ':' [expr]          (inclusive slices)
//   expr       := ['-'|'+'] term (('+'|'-') term)*  term := int ['*' ident] | ident ['*' int]
// Variables are resolved to binding slots at parse time, so evaluation is a handful of
// integer ops per index with no string lookups (the reference builds a std::map per call).
#pragma once

#include <string>
#include <vector>

#include "geometry.hpp"

namespace mtb {

enum class reduce_op : int32_t { plus = 0, times = 1, min = 2, max = 3 };
enum class access_kind : int32_t { read = 0, write = 1, readwrite = 2, reduce = 3 };
enum class binding_space : int32_t { global = 0, block = 1, local = 2 };

struct access_mode {
	access_kind kind = access_kind::read;
	reduce_op op = reduce_op::plus;
	bool reads() const { return kind == access_kind::read || kind == access_kind::readwrite; }
	bool writes() const { return kind == access_kind::write || kind == access_kind::readwrite; }
	bool reduces() const { return kind == access_kind::reduce; }
};

// constant + sum(coeff * var[slot]); duplicate variables are folded, zero terms dropped
struct lin_expr {
	int64_t constant = 0;
	struct term {
		int slot;
		int64_t coeff;
	};
	std::vector<term> terms; // first-occurrence order

	void add(int slot, int64_t coeff);
	span eval(const span* env) const;
};

struct index_expr {
	bool is_slice = false;
	bool has_lower = false, has_upper = false;
	lin_expr single, lower, upper;
	lin_expr lower_minus_upper; // folded lower-upper for the empty-slice test
};

struct access_decl {
	std::string argument;
	access_mode mode;
	std::vector<index_expr> indices;
};

struct var_binding {
	binding_space space = binding_space::global;
	int axis = 0; // grid axis this variable binds
	std::string name;
};

struct annotation {
	std::vector<var_binding> vars; // slot order
	std::vector<access_decl> accesses;

	const access_decl* find(const std::string& arg) const {
		for(const auto& a : accesses)
			if(a.argument == arg) return &a;
		return nullptr;
	}
};

annotation parse_annotation(const std::string& text);

// Evaluates one access of `ann` for a superblock; `domain` is the argument array's domain.
// Result is the half-open bounding box clipped to the domain (empty if a slice is empty
// for every thread). `env` must come from make_env.
box eval_access(const access_decl& acc, const span* env, const box& domain);

// Binding environment for a superblock (annotation.cpp:440-460 semantics).
void make_env(const annotation& ann, const box& superblock_threads, const point& block_size, span* env);

} // namespace mtb
