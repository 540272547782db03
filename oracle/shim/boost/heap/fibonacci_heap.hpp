// TEST INFRASTRUCTURE ONLY. Boost-free stand-in for the subset of
// boost::heap::fibonacci_heap that /root/reference/proj/core/src/serial_rbp.cpp
// uses (push -> handle, top, update(handle, value), empty), so the reference's
// serial RBP compiles into oracle/_ref without Boost.  The reference's
// comparator (PqLess, serial_rbp.cpp:19-24) is a strict total order on
// (residual, id), so any correct max-priority queue pops the same sequence.
#ifndef ORACLE_SHIM_BOOST_HEAP_FIBONACCI_HEAP_HPP
#define ORACLE_SHIM_BOOST_HEAP_FIBONACCI_HEAP_HPP

#include <cstdint>
#include <deque>
#include <set>

namespace boost {
namespace heap {

template <class Cmp>
struct compare {};

template <class T, class Option>
class fibonacci_heap;

template <class T, class Cmp>
class fibonacci_heap<T, compare<Cmp>> {
  struct Node {
    T value;
    uint64_t seq;
  };
  struct Order {
    bool operator()(const Node* a, const Node* b) const {
      Cmp less;
      if (less(a->value, b->value)) return true;
      if (less(b->value, a->value)) return false;
      return a->seq < b->seq;
    }
  };

 public:
  using handle_type = Node*;

  handle_type push(const T& v) {
    nodes_.push_back(Node{v, next_seq_++});
    Node* n = &nodes_.back();
    order_.insert(n);
    return n;
  }
  const T& top() const { return (*order_.rbegin())->value; }
  bool empty() const { return order_.empty(); }
  void pop() { order_.erase(std::prev(order_.end())); }
  void update(handle_type h, const T& v) {
    order_.erase(h);
    h->value = v;
    order_.insert(h);
  }

 private:
  std::deque<Node> nodes_;  // stable addresses
  std::set<Node*, Order> order_;
  uint64_t next_seq_ = 0;
};

}  // namespace heap
}  // namespace boost

#endif
