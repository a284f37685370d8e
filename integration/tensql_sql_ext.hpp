// tensql SQL frontend extension: ORDER BY and n-way joins.
//
// The reference frontend parses SELECT .. FROM t1 [JOIN t2 ON a = b | , t2]
// [WHERE ..] [GROUP BY ..] [LIMIT n] (sql_parser.cpp:46-79) and plans at most
// two tables (sql_planner.cpp:266-290); there is no ORDER BY (`order` is not
// even reserved, sql_parser.cpp:29-33), so TPC-H Q3 exists only as plan JSON.
// This header adds, on top of the unmodified library:
//
//   SELECT ... FROM t1 [JOIN t2 ON x = y [JOIN t3 ON u = v ...] | , t2, t3 ...]
//          [WHERE ...] [GROUP BY ...] [ORDER BY c [ASC|DESC], ...] [LIMIT n]
//
//   tensql::PlanPtr p = tqp_sqlx::parse_and_plan(sql, catalog);
//
// Statements the reference accepts (one or two tables, no ORDER BY) are
// handed to tensql::sql::parse_and_plan unchanged, so they plan exactly as
// before. ORDER BY becomes make_sort over the select list's output names
// (aliases), before LIMIT. With three or more tables the LAST table of the
// FROM list is the probe side and every prefix is the build side of the next
// join (t3 JOIN (t2 JOIN t1)): for a TPC-H chain written dimension-first
// (customer, orders, lineitem) this is the fact-probes-dimensions tree the
// fused B200 pipelines take (queries/q3.json's shape). Each table's own WHERE
// conjuncts are pushed below the joins, cross-table equalities join (from ON,
// or the first WHERE equality linking a table to the earlier ones), and the
// rest filters above the joins; the select list is planned as the reference
// planner does (aggregate slots, GROUP BY validity, literal coercion).
// Expressions are parsed by the reference parser itself (each clause is
// re-parsed as a one-table statement), so their syntax is the reference's.
#pragma once

#include <algorithm>
#include <cctype>
#include <optional>
#include <string>
#include <utility>
#include <variant>
#include <vector>

#include "tensql/plan.hpp"
#include "tensql/sql.hpp"
#include "tensql/strings.hpp"

namespace tqp_sqlx {

using tensql::sql::SqlError;
using tensql::sql::Token;
using tensql::sql::TokenKind;

inline bool kw(const Token& t, const char* w) {
  if (t.kind != TokenKind::Ident || t.text.size() != std::char_traits<char>::length(w)) return false;
  for (size_t i = 0; i < t.text.size(); ++i)
    if (std::tolower(static_cast<unsigned char>(t.text[i])) != w[i]) return false;
  return true;
}

struct OrderKey {
  std::string column;
  bool ascending = true;
  size_t offset = 0;
};

struct Statement {
  std::string select_sql;  // SELECT list text
  std::vector<std::pair<std::string, size_t>> tables;  // FROM list, in order
  std::vector<std::string> on;  // ON condition text per joined table (empty: comma join)
  std::string where, group_by;
  std::vector<OrderKey> order_by;
  std::optional<int64_t> limit;
  std::string core;  // the statement without ORDER BY / LIMIT (reference syntax)
};

// Splits the statement at its top-level clauses (token offsets into `sql`).
inline Statement split(const std::string& sql) {
  const std::vector<Token> tk = tensql::sql::tokenize(sql);
  Statement s;
  int depth = 0;
  // clause starts at paren depth 0
  std::vector<std::pair<std::string, size_t>> marks;  // (clause, token index)
  for (size_t i = 0; i < tk.size(); ++i) {
    if (tk[i].kind == TokenKind::LParen) ++depth;
    if (tk[i].kind == TokenKind::RParen) --depth;
    if (depth) continue;
    for (const char* c : {"select", "from", "join", "on", "where", "group", "order", "limit"})
      if (kw(tk[i], c)) marks.push_back({c, i});
  }
  auto text = [&](size_t a, size_t b) {  // tokens [a, b) as source text
    if (a >= b) return std::string();
    const size_t lo = tk[a].offset, hi = b < tk.size() ? tk[b].offset : sql.size();
    std::string t = sql.substr(lo, hi - lo);
    while (!t.empty() && std::isspace(static_cast<unsigned char>(t.back()))) t.pop_back();
    return t;
  };
  if (marks.empty() || marks[0].first != "select") throw SqlError("expected SELECT", 0);
  const size_t end = tk.size() - 1;  // the End token
  auto next_mark = [&](size_t m) { return m + 1 < marks.size() ? marks[m + 1].second : end; };
  size_t core_end = end;
  for (size_t m = 0; m < marks.size(); ++m) {
    const std::string& c = marks[m].first;
    const size_t a = marks[m].second + 1, b = next_mark(m);
    if (c == "select") {
      s.select_sql = text(a, b);
    } else if (c == "from" || c == "join") {
      // table [, table ...]
      for (size_t i = a; i < b; ++i) {
        if (tk[i].kind == TokenKind::Ident) s.tables.push_back({tk[i].text, tk[i].offset});
        else if (tk[i].kind != TokenKind::Comma) throw SqlError("expected a table name", tk[i].offset);
        if (c == "from" && tk[i].kind == TokenKind::Ident) s.on.push_back("");
      }
      if (c == "join") s.on.push_back("");
    } else if (c == "on") {
      if (s.on.empty()) throw SqlError("ON without JOIN", tk[marks[m].second].offset);
      s.on.back() = text(a, b);
    } else if (c == "where") {
      s.where = text(a, b);
    } else if (c == "group") {
      if (a >= b || !kw(tk[a], "by")) throw SqlError("expected BY after GROUP", tk[marks[m].second].offset);
      s.group_by = text(a + 1, b);
    } else if (c == "order") {
      if (a >= b || !kw(tk[a], "by")) throw SqlError("expected BY after ORDER", tk[marks[m].second].offset);
      core_end = std::min(core_end, marks[m].second);
      for (size_t i = a + 1; i < b;) {
        if (tk[i].kind != TokenKind::Ident) throw SqlError("expected a column name in ORDER BY", tk[i].offset);
        OrderKey k{tk[i].text, true, tk[i].offset};
        ++i;
        if (i < b && (kw(tk[i], "asc") || kw(tk[i], "desc"))) k.ascending = kw(tk[i++], "asc");
        s.order_by.push_back(k);
        if (i < b) {
          if (tk[i].kind != TokenKind::Comma) throw SqlError("expected ',' in ORDER BY", tk[i].offset);
          ++i;
        }
      }
      if (s.order_by.empty()) throw SqlError("empty ORDER BY", tk[marks[m].second].offset);
    } else if (c == "limit") {
      core_end = std::min(core_end, marks[m].second);
      if (b != a + 1 || tk[a].kind != TokenKind::Int) throw SqlError("expected a row count after LIMIT", tk[a].offset);
      s.limit = std::stoll(tk[a].text);
    }
  }
  if (s.tables.empty()) throw SqlError("expected FROM", end < tk.size() ? tk[end].offset : 0);
  s.on.resize(s.tables.size());
  s.core = text(0, core_end);
  return s;
}

namespace detail {

using namespace tensql;
using namespace tensql::sql;

struct Ctx {
  const Catalog& catalog;
  Schema schema;
  bool allow_aggs = false;
  std::vector<AggregateNode::Agg>* agg_out = nullptr;
  const Schema* agg_input = nullptr;
};

inline LogicalType type_of(const ExprPtr& e, const Ctx& c, size_t off) {
  try {
    return infer_expr_type(e, c.schema, c.catalog);
  } catch (const PlanError& err) {
    throw SqlError(err.what(), off);
  }
}
inline bool int_lit(const ExprPtr& e) {
  const auto* l = std::get_if<Literal>(&e->node);
  return l && l->type == LogicalType::Int64;
}
inline ExprPtr to_f64(ExprPtr e, LogicalType want) {  // an int literal against a float operand
  if (want == LogicalType::Float64 && int_lit(e))
    return lit_f64(static_cast<double>(std::get<int64_t>(std::get<Literal>(e->node).value)));
  return e;
}
inline void coerce(ExprPtr& l, ExprPtr& r, const Ctx& c, size_t off) {
  const LogicalType lt = type_of(l, c, off), rt = type_of(r, c, off);
  if (lt == rt) return;
  if (lt == LogicalType::Float64) r = to_f64(r, lt);
  if (rt == LogicalType::Float64) l = to_f64(l, rt);
}

// AST -> Expr with the reference planner's typing and coercion rules
// (sql_planner.cpp:49-168)
inline ExprPtr convert(const AstExprPtr& a, Ctx& c) {
  return std::visit(
      [&](const auto& x) -> ExprPtr {
        using T = std::decay_t<decltype(x)>;
        const size_t off = a->offset;
        if constexpr (std::is_same_v<T, AstCol>) {
          if (!schema_find(c.schema, x.name)) {
            if (c.agg_input && schema_find(*c.agg_input, x.name))
              throw SqlError("column '" + x.name + "' must appear in GROUP BY or inside an aggregate", off);
            throw SqlError("unknown column '" + x.name + "'", off);
          }
          return col(x.name);
        } else if constexpr (std::is_same_v<T, AstLit>) {
          return std::make_shared<const Expr>(Expr{Literal{x.type, x.value}});
        } else if constexpr (std::is_same_v<T, AstArith>) {
          ExprPtr l = convert(x.left, c), r = convert(x.right, c);
          coerce(l, r, c, off);
          if (x.op == ArithOp::DIV && int_lit(l) && int_lit(r)) {
            l = to_f64(l, LogicalType::Float64);
            r = to_f64(r, LogicalType::Float64);
          }
          ExprPtr e = make_arith(x.op, l, r);
          type_of(e, c, off);
          return e;
        } else if constexpr (std::is_same_v<T, AstCompare>) {
          ExprPtr l = convert(x.left, c), r = convert(x.right, c);
          coerce(l, r, c, off);
          ExprPtr e = make_compare(x.op, l, r);
          type_of(e, c, off);
          return e;
        } else if constexpr (std::is_same_v<T, AstLogical>) {
          ExprPtr e = make_logical(x.op, convert(x.left, c), convert(x.right, c));
          type_of(e, c, off);
          return e;
        } else if constexpr (std::is_same_v<T, AstNot>) {
          ExprPtr e = make_not(convert(x.input, c));
          type_of(e, c, off);
          return e;
        } else if constexpr (std::is_same_v<T, AstBetween>) {
          ExprPtr v = convert(x.input, c);
          const LogicalType vt = type_of(v, c, off);
          ExprPtr e = make_between(v, to_f64(convert(x.lo, c), vt), to_f64(convert(x.hi, c), vt));
          type_of(e, c, off);
          return e;
        } else if constexpr (std::is_same_v<T, AstCase>) {
          std::vector<CaseExpr::Branch> br;
          for (const auto& b : x.branches) br.push_back({convert(b.when, c), convert(b.then, c)});
          ExprPtr el = convert(x.else_value, c);
          bool f = type_of(el, c, off) == LogicalType::Float64;
          for (const auto& b : br) f = f || type_of(b.then, c, off) == LogicalType::Float64;
          if (f) {
            for (auto& b : br) b.then = to_f64(b.then, LogicalType::Float64);
            el = to_f64(el, LogicalType::Float64);
          }
          ExprPtr e = make_case(std::move(br), el);
          type_of(e, c, off);
          return e;
        } else if constexpr (std::is_same_v<T, AstLike>) {
          ExprPtr e = make_like(convert(x.input, c), x.pattern);
          type_of(e, c, off);
          return e;
        } else if constexpr (std::is_same_v<T, AstPredict>) {
          if (!c.catalog.find_model(x.model)) throw SqlError("unknown model '" + x.model + "'", off);
          std::vector<ExprPtr> args;
          for (const auto& arg : x.args) args.push_back(to_f64(convert(arg, c), LogicalType::Float64));
          ExprPtr e = make_predict(x.model, std::move(args));
          type_of(e, c, off);
          return e;
        } else if constexpr (std::is_same_v<T, AstAggCall>) {
          if (!c.allow_aggs || !c.agg_out) throw SqlError("aggregate functions are only allowed in the select list", off);
          Ctx ac{c.catalog, *c.agg_input};
          ExprPtr inner = x.star ? lit_i64(1) : convert(x.arg, ac);
          LogicalType out = type_of(inner, ac, off);
          if (x.fn == AggFn::Count) out = LogicalType::Int64;
          if (x.fn == AggFn::Avg) out = LogicalType::Float64;
          const std::string name = "$agg" + std::to_string(c.agg_out->size());
          c.agg_out->push_back({name, x.fn, inner});
          c.schema.push_back({name, out});
          return col(name);
        } else {
          throw SqlError("unsupported expression", off);
        }
      },
      a->node);
}

inline bool has_agg(const AstExprPtr& e) {
  if (!e) return false;
  return std::visit(
      [&](const auto& x) -> bool {
        using T = std::decay_t<decltype(x)>;
        if constexpr (std::is_same_v<T, AstAggCall>) return true;
        else if constexpr (std::is_same_v<T, AstArith> || std::is_same_v<T, AstCompare> || std::is_same_v<T, AstLogical>)
          return has_agg(x.left) || has_agg(x.right);
        else if constexpr (std::is_same_v<T, AstNot> || std::is_same_v<T, AstLike>) return has_agg(x.input);
        else if constexpr (std::is_same_v<T, AstBetween>) return has_agg(x.input) || has_agg(x.lo) || has_agg(x.hi);
        else if constexpr (std::is_same_v<T, AstCase>) {
          for (const auto& b : x.branches)
            if (has_agg(b.when) || has_agg(b.then)) return true;
          return has_agg(x.else_value);
        } else if constexpr (std::is_same_v<T, AstPredict>) {
          for (const auto& arg : x.args)
            if (has_agg(arg)) return true;
          return false;
        } else {
          return false;
        }
      },
      e->node);
}

inline void columns_of(const ExprPtr& e, std::vector<std::string>& out) {
  std::visit(
      [&](const auto& x) {
        using T = std::decay_t<decltype(x)>;
        if constexpr (std::is_same_v<T, ColRef>) out.push_back(x.name);
        else if constexpr (std::is_same_v<T, ArithExpr> || std::is_same_v<T, CompareExpr> || std::is_same_v<T, LogicalExpr>) {
          columns_of(x.left, out);
          columns_of(x.right, out);
        } else if constexpr (std::is_same_v<T, NotExpr> || std::is_same_v<T, LikeExpr>) {
          columns_of(x.input, out);
        } else if constexpr (std::is_same_v<T, BetweenExpr>) {
          columns_of(x.input, out);
          columns_of(x.lo, out);
          columns_of(x.hi, out);
        } else if constexpr (std::is_same_v<T, CaseExpr>) {
          for (const auto& b : x.branches) {
            columns_of(b.when, out);
            columns_of(b.then, out);
          }
          columns_of(x.else_value, out);
        } else if constexpr (std::is_same_v<T, PredictExpr>) {
          for (const auto& arg : x.args) columns_of(arg, out);
        }
      },
      e->node);
}

inline void conjuncts(const ExprPtr& e, std::vector<ExprPtr>& out) {
  if (const auto* lg = std::get_if<LogicalExpr>(&e->node); lg && lg->op == LogicalOp::AND) {
    conjuncts(lg->left, out);
    conjuncts(lg->right, out);
    return;
  }
  out.push_back(e);
}
inline ExprPtr and_all(const std::vector<ExprPtr>& v) {
  ExprPtr a = v[0];
  for (size_t i = 1; i < v.size(); ++i) a = make_logical(LogicalOp::AND, a, v[i]);
  return a;
}

// a clause re-parsed by the reference parser as a one-table statement
inline AstExprPtr parse_pred(const std::string& text, const std::string& table) {
  return tensql::sql::parse("SELECT 1 FROM " + table + " WHERE " + text).where;
}

// Three or more tables (see the header comment for the join tree).
inline PlanPtr plan_chain(const Statement& st, const Catalog& cat) {
  const size_t n = st.tables.size();
  std::vector<const TableSchema*> ts(n);
  Schema all;
  std::vector<int> owner;  // all[i] belongs to table owner[i]
  for (size_t i = 0; i < n; ++i) {
    ts[i] = cat.find_table(st.tables[i].first);
    if (!ts[i]) throw SqlError("unknown table '" + st.tables[i].first + "'", st.tables[i].second);
    for (size_t j = 0; j < i; ++j)
      if (iequals(st.tables[j].first, st.tables[i].first))
        throw SqlError("self-joins are not supported", st.tables[i].second);
    for (const auto& cs : *ts[i]) {
      if (schema_find(all, cs.name))
        throw SqlError("column '" + cs.name + "' exists in two tables; queries over ambiguous schemas are not supported",
                       st.tables[i].second);
      all.push_back(cs);
      owner.push_back(static_cast<int>(i));
    }
  }
  auto table_of = [&](const std::string& c) {
    for (size_t i = 0; i < all.size(); ++i)
      if (iequals(all[i].name, c)) return owner[i];
    return -1;
  };
  auto tables_of = [&](const ExprPtr& e) {
    std::vector<std::string> cs;
    columns_of(e, cs);
    std::vector<int> t;
    for (const auto& c : cs) t.push_back(table_of(c));
    std::sort(t.begin(), t.end());
    t.erase(std::unique(t.begin(), t.end()), t.end());
    return t;
  };
  Ctx wc{cat, all};
  const std::string& t0 = st.tables[0].first;
  std::vector<ExprPtr> conj;
  if (!st.where.empty()) {
    AstExprPtr w = parse_pred(st.where, t0);
    if (has_agg(w)) throw SqlError("aggregate functions are not allowed in WHERE", w->offset);
    conjuncts(convert(w, wc), conj);
  }
  // join keys: table i (i >= 1) joins the tables before it
  std::vector<std::pair<std::string, std::string>> keys(n);  // (key on table i, key on the prefix)
  std::vector<bool> have(n, false);
  auto eq_keys = [&](const ExprPtr& e, size_t i, std::pair<std::string, std::string>& k) {
    const auto* cmp = std::get_if<CompareExpr>(&e->node);
    if (!cmp || cmp->op != CompareOp::EQ) return false;
    const auto* l = std::get_if<ColRef>(&cmp->left->node);
    const auto* r = std::get_if<ColRef>(&cmp->right->node);
    if (!l || !r) return false;
    const int tl = table_of(l->name), tr = table_of(r->name);
    if (tl == static_cast<int>(i) && tr >= 0 && tr < static_cast<int>(i)) k = {l->name, r->name};
    else if (tr == static_cast<int>(i) && tl >= 0 && tl < static_cast<int>(i)) k = {r->name, l->name};
    else return false;
    return true;
  };
  for (size_t i = 1; i < n; ++i) {
    if (st.on[i].empty()) continue;
    AstExprPtr on = parse_pred(st.on[i], t0);
    if (!eq_keys(convert(on, wc), i, keys[i]))
      throw SqlError("JOIN ... ON must be a single equality between a column of the joined table and one of the tables "
                     "before it",
                     on->offset);
    have[i] = true;
  }
  std::vector<std::vector<ExprPtr>> side(n);
  std::vector<ExprPtr> residual;
  for (const auto& e : conj) {
    bool used = false;
    for (size_t i = 1; i < n && !used; ++i)
      if (!have[i] && eq_keys(e, i, keys[i])) used = have[i] = true;
    if (used) continue;
    const auto t = tables_of(e);
    if (t.size() == 1) side[t[0]].push_back(e);
    else if (t.empty()) side[0].push_back(e);  // constant conjuncts filter the first table
    else residual.push_back(e);
  }
  for (size_t i = 1; i < n; ++i)
    if (!have[i])
      throw SqlError("table '" + st.tables[i].first +
                         "' needs an equality with an earlier table (cross products are not supported)",
                     st.tables[i].second);
  auto scan = [&](size_t i) {
    PlanPtr p = make_scan(st.tables[i].first);
    if (!side[i].empty()) p = make_filter(p, and_all(side[i]));
    return p;
  };
  // the last table probes; every prefix is the build side of the next join
  PlanPtr root = scan(0);
  for (size_t i = 1; i < n; ++i) root = make_join(scan(i), root, keys[i].first, keys[i].second);
  if (!residual.empty()) root = make_filter(root, and_all(residual));

  // select list as the reference planner builds it (sql_planner.cpp:375-410)
  const Ast sel = tensql::sql::parse("SELECT " + st.select_sql + " FROM " + t0 +
                                     (st.group_by.empty() ? std::string() : " GROUP BY " + st.group_by));
  bool agg = !sel.group_by.empty();
  for (const auto& it : sel.select) agg = agg || has_agg(it.expr);
  std::vector<ProjectNode::Item> items;
  auto item_name = [](const SelectItem& it, size_t i) {
    if (it.alias) return *it.alias;
    if (const auto* c = std::get_if<AstCol>(&it.expr->node)) return c->name;
    return "_c" + std::to_string(i);
  };
  if (agg) {
    std::vector<std::string> gk;
    Schema post;
    for (const auto& [name, off] : sel.group_by) {
      const ColumnSpec* cs = schema_find(all, name);
      if (!cs) throw SqlError("unknown column '" + name + "'", off);
      gk.push_back(name);
      post.push_back(*cs);
    }
    std::vector<AggregateNode::Agg> aggs;
    Ctx sc{cat, post, true, &aggs, &all};
    for (size_t i = 0; i < sel.select.size(); ++i) {
      ExprPtr e = convert(sel.select[i].expr, sc);
      type_of(e, sc, sel.select[i].expr->offset);
      items.push_back({item_name(sel.select[i], i), e});
    }
    if (aggs.empty()) throw SqlError("grouped query needs at least one aggregate (DISTINCT is not supported)", 0);
    root = make_aggregate(root, std::move(gk), std::move(aggs));
  } else {
    Ctx sc{cat, all};
    for (size_t i = 0; i < sel.select.size(); ++i) items.push_back({item_name(sel.select[i], i), convert(sel.select[i].expr, sc)});
  }
  return make_project(root, std::move(items));
}

}  // namespace detail

// Parses and plans a statement (see the header comment).
inline tensql::PlanPtr parse_and_plan(const std::string& sql, const tensql::Catalog& catalog) {
  const Statement st = split(sql);
  tensql::PlanPtr p = st.tables.size() <= 2 ? tensql::sql::parse_and_plan(st.core, catalog)
                                            : detail::plan_chain(st, catalog);
  if (!st.order_by.empty()) {
    const tensql::Schema out = tensql::infer_schema(p, catalog);
    std::vector<tensql::SortNode::Key> keys;
    for (const auto& k : st.order_by) {
      const tensql::ColumnSpec* cs = tensql::schema_find(out, k.column);
      if (!cs) throw SqlError("ORDER BY column '" + k.column + "' is not in the select list", k.offset);
      keys.push_back({cs->name, k.ascending});
    }
    p = tensql::make_sort(p, std::move(keys));
  }
  if (st.limit) p = tensql::make_limit(p, *st.limit);
  return p;
}

}  // namespace tqp_sqlx
