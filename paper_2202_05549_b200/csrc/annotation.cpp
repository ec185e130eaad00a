#include "annotation.hpp"

#include <cctype>

namespace mtb {

void lin_expr::add(int slot, int64_t coeff) {
	for(size_t i = 0; i < terms.size(); ++i) {
		if(terms[i].slot != slot) continue;
		terms[i].coeff += coeff;
		if(terms[i].coeff == 0) terms.erase(terms.begin() + static_cast<std::ptrdiff_t>(i));
		return;
	}
	if(coeff != 0) terms.push_back({slot, coeff});
}

span lin_expr::eval(const span* env) const {
	span acc{constant, constant};
	for(const auto& t : terms) acc = span::sum(acc, span::scaled(t.coeff, env[t.slot]));
	return acc;
}

namespace {

enum class tok { ident, number, sym, end };

struct token {
	tok kind = tok::end;
	std::string text;
	int64_t value = 0;
	int line = 1, col = 1;
};

// Single-pass tokenizer; positions are 1-based line/column of the token start.
class scanner {
  public:
	explicit scanner(const std::string& s) : src_(s) { step(); }
	const token& cur() const { return cur_; }
	token take() {
		token t = cur_;
		step();
		return t;
	}

  private:
	const std::string& src_;
	size_t at_ = 0;
	int line_ = 1, col_ = 1;
	token cur_;

	char ch(size_t off = 0) const { return at_ + off < src_.size() ? src_[at_ + off] : '\0'; }
	void bump() {
		if(src_[at_] == '\n') {
			++line_;
			col_ = 1;
		} else {
			++col_;
		}
		++at_;
	}
	void step() {
		while(at_ < src_.size() && std::isspace(static_cast<unsigned char>(src_[at_]))) bump();
		cur_ = token{};
		cur_.line = line_;
		cur_.col = col_;
		if(at_ >= src_.size()) {
			cur_.kind = tok::end;
			cur_.text = "<end of input>";
			return;
		}
		const unsigned char c = static_cast<unsigned char>(ch());
		if(std::isalpha(c) || c == '_') {
			cur_.kind = tok::ident;
			while(at_ < src_.size() && (std::isalnum(static_cast<unsigned char>(ch())) || ch() == '_')) {
				cur_.text.push_back(ch());
				bump();
			}
			return;
		}
		if(std::isdigit(c)) {
			cur_.kind = tok::number;
			while(at_ < src_.size() && std::isdigit(static_cast<unsigned char>(ch()))) {
				cur_.text.push_back(ch());
				if(__builtin_mul_overflow(cur_.value, int64_t{10}, &cur_.value) || __builtin_add_overflow(cur_.value, int64_t{ch() - '0'}, &cur_.value))
					throw parse_error(cur_.line, cur_.col, "integer literal too large");
				bump();
			}
			return;
		}
		cur_.kind = tok::sym;
		if(c == '=' && ch(1) == '>') {
			cur_.text = "=>";
			bump();
			bump();
			return;
		}
		static const std::string singles = "[](),:+-*";
		if(singles.find(static_cast<char>(c)) == std::string::npos)
			throw parse_error(line_, col_, std::string("unexpected character '") + static_cast<char>(c) + "'");
		cur_.text = std::string(1, static_cast<char>(c));
		bump();
	}
};

class reader {
  public:
	explicit reader(const std::string& text) : in_(text) {}

	annotation run() {
		binding();
		while(at_sym(",")) {
			in_.take();
			binding();
		}
		want_sym("=>");
		if(in_.cur().kind != tok::end) {
			access();
			while(at_sym(",")) {
				in_.take();
				access();
			}
		}
		if(in_.cur().kind != tok::end) die(in_.cur(), "expected end of annotation, got \"" + in_.cur().text + "\"");
		return std::move(ann_);
	}

  private:
	scanner in_;
	annotation ann_;

	[[noreturn]] static void die(const token& t, const std::string& msg) { throw parse_error(t.line, t.col, msg); }
	bool at_sym(const char* s) const { return in_.cur().kind == tok::sym && in_.cur().text == s; }
	token want_sym(const char* s) {
		if(!at_sym(s)) die(in_.cur(), std::string("expected \"") + s + "\", got \"" + in_.cur().text + "\"");
		return in_.take();
	}
	token want_ident() {
		if(in_.cur().kind != tok::ident) die(in_.cur(), "expected identifier, got \"" + in_.cur().text + "\"");
		return in_.take();
	}
	int slot_of(const std::string& name) const {
		for(size_t i = 0; i < ann_.vars.size(); ++i)
			if(ann_.vars[i].name == name) return static_cast<int>(i);
		return -1;
	}
	void declare(const token& t, binding_space space, int axis) {
		if(slot_of(t.text) >= 0) die(t, "duplicate variable \"" + t.text + "\"");
		ann_.vars.push_back({space, axis, t.text});
	}

	void binding() {
		const token sp = want_ident();
		binding_space space;
		if(sp.text == "global")
			space = binding_space::global;
		else if(sp.text == "block")
			space = binding_space::block;
		else if(sp.text == "local")
			space = binding_space::local;
		else
			die(sp, "expected binding space (global, block or local), got \"" + sp.text + "\"");
		int count = 0;
		if(at_sym("[")) {
			in_.take();
			for(;;) {
				declare(want_ident(), space, count++);
				if(at_sym("]")) {
					in_.take();
					break;
				}
				want_sym(",");
			}
		} else {
			declare(want_ident(), space, count++);
		}
		if(count > kMaxRank) die(sp, "a binding may name at most 3 variables");
	}

	void access() {
		const token m = want_ident();
		access_decl a;
		if(m.text == "read") {
			a.mode.kind = access_kind::read;
		} else if(m.text == "write") {
			a.mode.kind = access_kind::write;
		} else if(m.text == "readwrite") {
			a.mode.kind = access_kind::readwrite;
		} else if(m.text == "reduce") {
			a.mode.kind = access_kind::reduce;
			want_sym("(");
			const token op = in_.take();
			if(op.kind == tok::sym && op.text == "+")
				a.mode.op = reduce_op::plus;
			else if(op.kind == tok::sym && op.text == "*")
				a.mode.op = reduce_op::times;
			else if(op.kind == tok::ident && op.text == "min")
				a.mode.op = reduce_op::min;
			else if(op.kind == tok::ident && op.text == "max")
				a.mode.op = reduce_op::max;
			else
				die(op, "reduce operator must be +, *, min or max");
			want_sym(")");
		} else {
			die(m, "expected access mode (read, write, readwrite or reduce), got \"" + m.text + "\"");
		}
		const token arg = want_ident();
		a.argument = arg.text;
		if(ann_.find(a.argument)) die(arg, "duplicate argument \"" + a.argument + "\"");
		want_sym("[");
		for(;;) {
			a.indices.push_back(index());
			if(at_sym("]")) {
				in_.take();
				break;
			}
			want_sym(",");
		}
		if(a.indices.size() > static_cast<size_t>(kMaxRank)) die(arg, "arrays have at most 3 axes");
		ann_.accesses.push_back(std::move(a));
	}

	index_expr index() {
		index_expr ix;
		if(!at_sym(":")) {
			ix.lower = expr();
			ix.has_lower = true;
		}
		if(!at_sym(":")) {
			ix.single = ix.lower;
			return ix;
		}
		in_.take();
		ix.is_slice = true;
		if(!at_sym("]") && !at_sym(",")) {
			ix.upper = expr();
			ix.has_upper = true;
		}
		if(ix.has_lower && ix.has_upper) {
			ix.lower_minus_upper = ix.lower;
			ix.lower_minus_upper.constant -= ix.upper.constant;
			for(const auto& t : ix.upper.terms) ix.lower_minus_upper.add(t.slot, -t.coeff);
		}
		return ix;
	}

	lin_expr expr() {
		lin_expr e;
		int64_t sign = 1;
		if(at_sym("-")) {
			in_.take();
			sign = -1;
		} else if(at_sym("+")) {
			in_.take();
		}
		term(e, sign);
		while(at_sym("+") || at_sym("-")) {
			sign = in_.take().text == "+" ? 1 : -1;
			term(e, sign);
		}
		return e;
	}

	int bound_slot(const token& v) const {
		const int s = slot_of(v.text);
		if(s < 0) die(v, "unbound variable \"" + v.text + "\"");
		return s;
	}

	void term(lin_expr& e, int64_t sign) {
		const token t = in_.cur();
		if(t.kind == tok::number) {
			const token lit = in_.take();
			if(!at_sym("*")) {
				e.constant += sign * lit.value;
				return;
			}
			const token star = in_.take();
			if(in_.cur().kind == tok::number) die(star, "constant products are not index expressions");
			const token v = want_ident();
			e.add(bound_slot(v), sign * lit.value);
			return;
		}
		if(t.kind == tok::ident) {
			const token v = in_.take();
			const int s = bound_slot(v);
			if(!at_sym("*")) {
				e.add(s, sign);
				return;
			}
			const token star = in_.take();
			if(in_.cur().kind == tok::ident) die(star, "nonlinear expression: product of variables \"" + v.text + "\" and \"" + in_.cur().text + "\"");
			if(in_.cur().kind != tok::number) die(star, "expected integer coefficient after \"*\"");
			e.add(s, sign * in_.take().value);
			return;
		}
		die(t, "expected index expression, got \"" + t.text + "\"");
	}
};

} // namespace

annotation parse_annotation(const std::string& text) { return reader(text).run(); }

void make_env(const annotation& ann, const box& sb, const point& bs, span* env) {
	for(size_t i = 0; i < ann.vars.size(); ++i) {
		const auto& v = ann.vars[i];
		if(v.axis >= sb.rank()) throw validation_error("binding names more variables than the launch grid has axes");
		const int k = v.axis;
		switch(v.space) {
		case binding_space::global: env[i] = {sb.lo[k], sb.hi[k] - 1}; break;
		case binding_space::block: env[i] = {sb.lo[k] / bs[k], (sb.hi[k] - 1) / bs[k]}; break;
		case binding_space::local: env[i] = {0, bs[k] - 1}; break;
		}
	}
}

box eval_access(const access_decl& acc, const span* env, const box& domain) {
	const int rank = domain.rank();
	if(static_cast<int>(acc.indices.size()) != rank)
		throw validation_error("argument \"" + acc.argument + "\" is indexed with " + std::to_string(acc.indices.size()) + " axes but has rank "
		                       + std::to_string(rank));
	box r;
	r.lo = point::zeros(rank);
	r.hi = point::zeros(rank);
	for(int k = 0; k < rank; ++k) {
		const auto& ix = acc.indices[static_cast<size_t>(k)];
		span s;
		if(!ix.is_slice) {
			s = ix.single.eval(env);
		} else {
			s.lo = ix.has_lower ? ix.lower.eval(env).lo : domain.lo[k];
			s.hi = ix.has_upper ? ix.upper.eval(env).hi : domain.hi[k] - 1;
			if(ix.has_lower && ix.has_upper && ix.lower_minus_upper.eval(env).lo > 0) s = span{};
		}
		if(s.is_empty()) return box::empty(rank);
		// inclusive -> half-open, clipped to the domain
		r.lo[k] = std::max(s.lo, domain.lo[k]);
		r.hi[k] = std::min(s.hi + 1, domain.hi[k]);
		if(r.hi[k] <= r.lo[k]) return box::empty(rank);
	}
	return r;
}

} // namespace mtb
